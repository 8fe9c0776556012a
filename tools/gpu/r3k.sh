#!/bin/bash
# x gathers with / without the L2 evict-last policy on the c5 headline layout (ELL-8, C = 64), alternating.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/time_launches.py c5 ELL --index16 2 --reps 10 1024,64,0,64 1024,64,0,262208 1024,128,0,64 1024,128,0,262208 1024,64,0,64 1024,64,0,262208 512,64,0,64 512,64,0,262208 > gpurun_out/r3k_tl.log 2>&1
timeout 600 python tools/time_launches.py c2 ELL --index16 2 --reps 50 1024,64,25,64 1024,64,25,262208 1024,64,25,64 1024,64,25,262208 128,64,25,65600 128,64,25,327744 >> gpurun_out/r3k_tl.log 2>&1
cat gpurun_out/r3k_tl.log
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --profile-from-start off -c 2 --csv python tools/kernel_one.py c2 ELL 1 --index16 2 --launch 1024,64,25,262208 > gpurun_out/r3k_ncu_c2.csv 2>&1; grep -E "dram__|inst_exec|duration" gpurun_out/r3k_ncu_c2.csv | cut -d, -f5,13-15 | tail -n 4
