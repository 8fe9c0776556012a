#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/time_launches.py c2 COO --reps 50 128,255,-1,8 128,255,-1,0x120 256,255,-1,0x120 64,255,-1,0x120 256,128,-1,0x110 > gpurun_out/r2k_tl.log 2>&1
timeout 600 python tools/time_launches.py c2 CSR --csr-alg 3 --reps 50 128,255,-1,0x220 256,255,-1,0x220 64,255,-1,0x220 128,255,-1,0x120 256,255,-1,0x120 >> gpurun_out/r2k_tl.log 2>&1
timeout 600 python tools/time_launches.py c3 CSR --csr-alg 3 --reps 20 128,255,-1,0x220 256,255,-1,0x220 128,255,-1,0x120 128,32,50,0x104 >> gpurun_out/r2k_tl.log 2>&1
timeout 600 python tools/time_launches.py c3 COO --reps 20 64,64,0,8 128,255,-1,0x120 256,255,-1,0x120 >> gpurun_out/r2k_tl.log 2>&1
cat gpurun_out/r2k_tl.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_gputests.log 2>&1; tail -n 3 gpurun_out/r2k_gputests.log
