#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "launch_variants or spmv_all or csr" > gpurun_out/r4f_tests.log 2>&1; tail -n 2 gpurun_out/r4f_tests.log
grep -E "assert|Error" gpurun_out/r4f_tests.log | head -5
T=gpurun_out/r4f_tl.log
timeout 600 python tools/time_launches.py c2 CSR --csr-alg 2 --reps 20 256,64,0,16 256,128,0,272 256,128,0,264 128,128,0,272 512,128,0,272 256,255,0,288 > $T 2>&1
timeout 600 python tools/time_launches.py c4 CSR --csr-alg 2 --reps 10 256,255,0,16 256,128,0,272 256,128,0,264 128,128,0,272 256,255,0,288 >> $T 2>&1
cat $T
timeout 900 python tools/format_sweep.py --configs band64_2M,c2,c4 --formats CSR-vector --out gpurun_out/r4f_sweep > gpurun_out/r4f.log 2>&1; tail -n 3 gpurun_out/r4f_sweep.md
