#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "launch_variants or determinism or coo" > gpurun_out/r4e_tests.log 2>&1; tail -n 2 gpurun_out/r4e_tests.log
T=gpurun_out/r4e_tl.log
timeout 600 python tools/time_launches.py c2 COO --reps 20 128,64,25,8 128,128,25,16 256,128,25,16 64,128,25,16 128,255,25,16 64,255,0,16 > $T 2>&1
timeout 600 python tools/time_launches.py c3 COO --reps 10 64,255,0,8 64,128,0,16 128,128,0,16 64,255,0,16 >> $T 2>&1
cat $T
timeout 900 python tools/ncu_traffic.py c3 COO CSR-merge --launch "COO=64,255,0,8;CSR-merge=64,255,0,2056" --out gpurun_out/r4e_traffic_c3.json > gpurun_out/r4e_traffic.log 2>&1; tail -n 2 gpurun_out/r4e_traffic.log | cut -c1-300
