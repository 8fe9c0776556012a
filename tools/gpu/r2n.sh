#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 1800 python bench.py ) > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2n_bench.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ['value','ms_per_step','step_phases_ms','steps_ms','clocks','e2e','mflops_per_w','gpu_launches']}); print(d['config']); print(d['roofline'])
print({c: (v.get('format'), v.get('kernel_us'), v.get('frac_measured_peak'), v.get('frac_gather_ceiling'), v.get('leg_seconds')) for c, v in d.get('per_config', {}).items()}); print(d['cpu_baseline'])"
tail -n 3 gpurun_out/r2n_bench.err
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" --csv --log-file gpurun_out/r2n_launches.csv python bench.py --steps 1 --warmup 1 --per-config none --no-cpu-baseline --no-e2e > gpurun_out/r2n_ncu_bench.log 2>&1
tail -n 2 gpurun_out/r2n_ncu_bench.log; wc -l gpurun_out/r2n_launches.csv
