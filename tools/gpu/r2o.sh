#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_index16_predict.py -x -q > gpurun_out/r2o_tests.log 2>&1; tail -n 3 gpurun_out/r2o_tests.log
timeout 600 python tools/time_launches.py c3 COO --reps 20 64,64,0,8 64,64,0,0x408 128,64,0,0x408 256,64,0,0x408 128,128,0,0x404 256,128,0,0x404 64,255,0,0x408 512,64,0,0x408 > gpurun_out/r2o_tl.log 2>&1
timeout 600 python tools/time_launches.py c2 COO --reps 50 128,64,0,8 128,64,0,0x408 256,64,0,0x408 256,128,0,0x404 >> gpurun_out/r2o_tl.log 2>&1
timeout 600 python tools/time_launches.py c4 COO --reps 20 64,32,0,4 64,64,0,0x408 128,64,0,0x408 256,128,0,0x404 >> gpurun_out/r2o_tl.log 2>&1
cat gpurun_out/r2o_tl.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dict_flags -c 1 --csv python tools/kernel_one.py c5 ELL 1 --index16 2 --launch 1024,128,0,65600 2>&1 | grep -E "k_dict|duration" | tail -n 2
