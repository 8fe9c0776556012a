#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "nnz_split or launch_variants" > gpurun_out/r3r_tests.log 2>&1; tail -n 3 gpurun_out/r3r_tests.log
grep -E "Error|assert" gpurun_out/r3r_tests.log | head -5
L=""
for b in 64 128 256; do for r in 32 64 128; do L="$L $b,$r,-1,0x808"; done; done
timeout 600 python tools/time_launches.py c3 CSR --csr-alg 3 --reps 10 64,64,-1,0x408 $L > gpurun_out/r3r_tl.log 2>&1
timeout 300 python tools/time_launches.py c3 COO --reps 10 64,64,0,8 128,64,0,8 >> gpurun_out/r3r_tl.log 2>&1
timeout 600 python tools/time_launches.py c4 CSR --csr-alg 3 --reps 10 256,32,-1,0x404 $L >> gpurun_out/r3r_tl.log 2>&1
timeout 600 python tools/time_launches.py c2 CSR --csr-alg 3 --reps 10 128,128,100,528 $L >> gpurun_out/r3r_tl.log 2>&1
cat gpurun_out/r3r_tl.log
