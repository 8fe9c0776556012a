#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/r2i_c5_ell8 python tools/kernel_one.py c5 ELL 1 --index16 2 --launch 1024,255,0,65600 > gpurun_out/r2i_ncu_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/r2i_c5_ell32 python tools/kernel_one.py c5 ELL 1 --index16 0 --launch 256,64,0,65664 > gpurun_out/r2i_ncu_c5b.log 2>&1
tail -2 gpurun_out/r2i_ncu_c5.log gpurun_out/r2i_ncu_c5b.log
( time timeout 1500 python bench.py ) > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2i_bench.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ['value','ms_per_step','step_phases_ms','steps_ms','clocks','e2e','mflops_per_w']}); print(d['config']); print(d['roofline'])
print({c: (v.get('format'), v.get('kernel_us'), v.get('frac_measured_peak'), v.get('frac_gather_ceiling'), v.get('leg_seconds')) for c, v in d.get('per_config', {}).items()})"
tail -3 gpurun_out/r2i_bench.err
