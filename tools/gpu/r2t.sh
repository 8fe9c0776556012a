#!/bin/bash
# Round-2 re-entry check: full GPU suite, smoke, default bench on current HEAD.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2t_smi.txt 2>&1
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/r2t_tests.log 2>&1; tail -n 3 gpurun_out/r2t_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1; tail -n 2 gpurun_out/r2t_smoke.log
timeout 1200 python bench.py > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; tail -c 3000 gpurun_out/r2t_bench.json; tail -n 5 gpurun_out/r2t_bench.err
