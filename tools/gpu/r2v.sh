#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coo_stream or determinism or launch_variants" > gpurun_out/r2v_new.log 2>&1; tail -n 15 gpurun_out/r2v_new.log
T=gpurun_out/r2v_tl.log
L=""
for b in 64 128 256; do for e in 16 24 32; do for r in 128 255; do L="$L $b,$r,-1,$((0x200+e))"; done; done; done
timeout 600 python tools/time_launches.py c2 COO --reps 50 128,64,0,8 $L > $T 2>&1
L=""
for b in 64 128 256; do for e in 8 16 24; do for r in 128 255; do L="$L $b,$r,-1,$((0x200+e))"; done; done; done
timeout 600 python tools/time_launches.py c3 COO --reps 20 64,64,0,8 $L >> $T 2>&1
timeout 600 python tools/time_launches.py c3 HYB --reps 20 64,64,25,8 $L >> $T 2>&1
L=""
for b in 64 128 256; do for e in 16 32; do for r in 128 255; do L="$L $b,$r,-1,$((0x200+e))"; done; done; done
timeout 600 python tools/time_launches.py c4 COO --reps 20 64,32,0,4 $L >> $T 2>&1
cat $T
