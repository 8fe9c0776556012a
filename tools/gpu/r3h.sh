#!/bin/bash
# release_csr + pad-code table trick + e2e with two steps in flight on c5: parity, then the default bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_index16_predict.py -x -q > gpurun_out/r3h_tests.log 2>&1; tail -n 2 gpurun_out/r3h_tests.log
timeout 1500 python bench.py > gpurun_out/r3h_bench.json 2> gpurun_out/r3h_bench.err; tail -n 3 gpurun_out/r3h_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r3h_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['steps_ms'], d['roofline']['frac'], d['roofline']['kernel_avg_us'], d['clocks'], d['config']['launch'])
print(d['e2e']); print(d['energy'], d['mflops_per_w'])
for c,v in d['per_config'].items(): print(c, {k:v.get(k) for k in ['format','launch','kernel_us','frac_measured_peak','frac_gather_ceiling']})
print(d['cpu_baseline']['value'], d['cpu_baseline'].get('cores'))"
