#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py -x -q -k "release or graph or plan_matches" > gpurun_out/r3i_tests.log 2>&1; tail -n 3 gpurun_out/r3i_tests.log
grep -E "Error|error|assert" gpurun_out/r3i_tests.log | head -20
timeout 900 python bench.py --config c2 --per-config c1 --no-cpu-baseline --steps 3 > gpurun_out/r3i_bench.json 2> gpurun_out/r3i_bench.err; tail -n 2 gpurun_out/r3i_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r3i_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['per_config'], d['e2e'])"
