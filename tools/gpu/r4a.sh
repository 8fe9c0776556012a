#!/bin/bash
# 256-bit evict-first stream loads: parity of the touched kernels, then timings.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_index16_predict.py -x -q -k "launch_variants or nnz_split or coo or sliced or layouts or index16 or 8 or ell or sell" > gpurun_out/r4a_tests.log 2>&1; tail -n 2 gpurun_out/r4a_tests.log
T=gpurun_out/r4a_tl.log
timeout 600 python tools/time_launches.py c3 COO --reps 10 64,64,0,8 128,64,0,8 64,128,0,8 > $T 2>&1
timeout 600 python tools/time_launches.py c3 CSR --csr-alg 3 --reps 10 64,64,-1,0x808 128,64,-1,0x808 64,128,-1,0x808 >> $T 2>&1
timeout 600 python tools/time_launches.py c2 COO --reps 20 128,64,0,8 64,64,0,8 256,64,0,8 >> $T 2>&1
timeout 900 python tools/time_launches.py c5 ELL --index16 2 --reps 10 1024,64,0,64 1024,64,0,128 512,64,0,128 1024,64,0,65664 512,128,0,128 1024,64,0,64 >> $T 2>&1
timeout 600 python tools/time_launches.py c2 ELL --index16 2 --reps 50 1024,64,25,64 1024,64,25,128 512,128,25,128 >> $T 2>&1
timeout 600 python tools/time_launches.py c4 SELL --reps 20 256,255,0,65600 256,255,0,65664 128,128,0,64 >> $T 2>&1
cat $T
