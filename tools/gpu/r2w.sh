#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_coo -c 2 -o gpurun_out/r2w_coostream python tools/kernel_one.py c2 COO 2 --launch 256,128,-1,528 > gpurun_out/r2w.log 2>&1
tail -3 gpurun_out/r2w.log
