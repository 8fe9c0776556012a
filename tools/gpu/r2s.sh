#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
A="--per-config none --no-cpu-baseline --no-e2e --steps 8"
timeout 900 python bench.py $A > gpurun_out/r2s_a.json 2> gpurun_out/r2s_a.err
python -c "
import json; d=json.loads(open('gpurun_out/r2s_a.json').read().strip().splitlines()[-1])
print('a', d['value'], d['steps_ms'], d['clocks'], d['config']['launch'], d['roofline']['kernel_avg_us']); print(d['steps_phase_ms'])"
tail -n 3 gpurun_out/r2s_a.err
