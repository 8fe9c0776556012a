#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_index16_predict.py tests/test_gpu_plan.py -x -q > gpurun_out/r2p_tests.log 2>&1; tail -n 3 gpurun_out/r2p_tests.log
L="1024,64,0,65600 1024,128,0,65600 512,64,0,65664 1024,64,0,65664 256,64,0,65664 256,64,0,65600 512,64,0,65600"
timeout 900 python tools/time_launches.py c5 ELL --index16 2 --reps 10 $L > gpurun_out/r2p_tl.log 2>&1
timeout 900 python tools/time_launches.py c5 ELL --index16 0 --reps 10 256,64,0,65664 1024,64,0,65600 512,64,0,65664 >> gpurun_out/r2p_tl.log 2>&1
timeout 600 python tools/time_launches.py c2 ELL --index16 2 --reps 50 1024,64,0,65600 128,64,25,65600 512,64,0,65600 >> gpurun_out/r2p_tl.log 2>&1
timeout 600 python tools/time_launches.py c2 ELL --index16 1 --reps 50 1024,64,0,64 1024,64,0,65600 >> gpurun_out/r2p_tl.log 2>&1
timeout 600 python tools/time_launches.py c2 ELL --index16 0 --reps 50 1024,64,0,65600 256,64,0,65600 >> gpurun_out/r2p_tl.log 2>&1
cat gpurun_out/r2p_tl.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dict_flags -c 1 --csv python tools/kernel_one.py c5 ELL 1 --index16 2 --launch 1024,128,0,65600 2>&1 | grep -E "k_dict" | tail -n 1
