#!/bin/bash
# r2 session B: smoke, default bench (c5 + per_config + cpu leg), virtual ranks, predict tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/r2b_smoke.log 2>&1
( time timeout 1500 python bench.py ) > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
( time timeout 600 python bench.py --gpus 4 --virtual --config c2 --no-cpu-baseline --per-config none ) > gpurun_out/r2b_virtual4.json 2> gpurun_out/r2b_virtual4.err
timeout 1500 python -m pytest tests/test_gpu_bench_multirank.py tests/test_gpu_index16_predict.py -x -q > gpurun_out/r2b_tests.log 2>&1
tail -3 gpurun_out/r2b_smoke.log; tail -c 3000 gpurun_out/r2b_bench.json; tail -5 gpurun_out/r2b_bench.err; tail -c 1500 gpurun_out/r2b_virtual4.json; tail -5 gpurun_out/r2b_virtual4.err; tail -5 gpurun_out/r2b_tests.log
