#!/bin/bash
# Session-3 final validation: full GPU suite, smoke, default bench (c5 headline + c1..c4 + CPU oracle + e2e).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/r4g_tests.log 2>&1; tail -n 3 gpurun_out/r4g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4g_smoke.log 2>&1; tail -n 1 gpurun_out/r4g_smoke.log
timeout 1500 python bench.py > gpurun_out/r4g_bench.json 2> gpurun_out/r4g_bench.err; tail -n 3 gpurun_out/r4g_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r4g_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['steps_ms'], d['roofline'], d['clocks'], d['step_phases_ms'])
print(d['e2e']); print(d['energy'], d['mflops_per_w'], d['gpu_launches'])
for c,v in d['per_config'].items(): print(c, {k:v.get(k) for k in ['format','launch','kernel_us','frac_measured_peak','frac_gather_ceiling','us_per_step_graph','us_per_step_eager']})
print(d['cpu_baseline']['value'], d['cpu_baseline'].get('cores'))"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r4g_ref.json 2> gpurun_out/r4g_ref.err; tail -c 400 gpurun_out/r4g_ref.json
