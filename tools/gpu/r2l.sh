#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,power.draw,power.limit,temperature.gpu --format=csv > gpurun_out/r2l_smi.txt
timeout 600 python tools/power_probe.py c5 ELL 2 --launch 512,64,0,65664 > gpurun_out/r2l_probe.log 2>&1
timeout 600 python tools/power_probe.py c5 ELL 2 --launch 1024,255,0,65600 >> gpurun_out/r2l_probe.log 2>&1
timeout 600 python tools/power_probe.py c5 ELL 0 --launch 256,64,0,65664 >> gpurun_out/r2l_probe.log 2>&1
timeout 600 python tools/power_probe.py c2 SELL 2 --launch 1024,128,0,65600 --E 100 >> gpurun_out/r2l_probe.log 2>&1
cat gpurun_out/r2l_probe.log; cat gpurun_out/r2l_smi.txt
