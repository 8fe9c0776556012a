#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=""
for b in 64 128 256 512; do for c in -1 50 100; do for k in 4 8 16; do L="$L $b,64,$c,$k"; done; done; done
timeout 900 python tools/time_launches.py c3 CSR --csr-alg 3 --reps 10 $L 128,128,100,8 256,128,100,8 128,255,100,16 > gpurun_out/r2z_tl.log 2>&1
cat gpurun_out/r2z_tl.log
