#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L="1024,255,0,65600 1024,64,0,65600 512,64,0,65600 256,64,0,65600 256,64,0,65664 1024,64,0,65664 512,128,0,65664 1024,64,0,65792 512,128,0,65792 256,255,0,65792 1024,64,0,64 1024,64,0,128 1024,64,0,256"
timeout 900 python tools/time_launches.py c5 ELL --index16 2 --reps 10 $L > gpurun_out/r2h_tl.log 2>&1
timeout 900 python tools/time_launches.py c5 ELL --index16 0 --reps 10 256,64,0,65664 1024,64,0,65664 1024,64,0,65792 512,128,0,65600 >> gpurun_out/r2h_tl.log 2>&1
cat gpurun_out/r2h_tl.log
