#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/alloc_churn.py c5 ELL 2 --launch 512,64,0,65600 > gpurun_out/r2g_churn.log 2>&1
timeout 600 python tools/alloc_churn.py c5 ELL 2 --launch 512,64,0,65600 --trim >> gpurun_out/r2g_churn.log 2>&1
timeout 600 python tools/alloc_churn.py c5 ELL 0 --launch 256,64,0,65664 >> gpurun_out/r2g_churn.log 2>&1
cat gpurun_out/r2g_churn.log | tail -5
