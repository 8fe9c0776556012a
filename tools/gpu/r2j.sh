#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_index16_predict.py -x -q > gpurun_out/r2j_tests.log 2>&1; tail -2 gpurun_out/r2j_tests.log
L="1024,255,0,65600 1024,255,0,196672 1024,64,0,196672 512,64,0,65664 512,64,0,196736 1024,64,0,196736 512,128,0,196672 256,128,0,196736 1024,255,0,196640"
timeout 900 python tools/time_launches.py c5 ELL --index16 2 --reps 10 $L > gpurun_out/r2j_tl.log 2>&1
timeout 600 python tools/time_launches.py c2 ELL --index16 2 --reps 50 1024,64,0,65600 1024,64,0,196672 512,64,0,196672 1024,64,0,196736 128,64,25,65600 >> gpurun_out/r2j_tl.log 2>&1
cat gpurun_out/r2j_tl.log
for tool in memcheck racecheck synccheck; do timeout 1200 compute-sanitizer --tool $tool python tools/sanitize_cases.py ragged_empty,long_rows,rmat10,mixed_tiles > gpurun_out/r2j_san_$tool.log 2>&1; tail -2 gpurun_out/r2j_san_$tool.log; done
