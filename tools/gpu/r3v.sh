#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_index16_predict.py tests/test_selector.py -x -q -k "tune or predict or gate or select" > gpurun_out/r3v_tests.log 2>&1; tail -n 2 gpurun_out/r3v_tests.log
timeout 900 python bench.py --per-config none --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/r3v_bench.json 2> gpurun_out/r3v_bench.err; tail -n 2 gpurun_out/r3v_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r3v_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['steps_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['step_phases_ms'], d['config']['format'])"
