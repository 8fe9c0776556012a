#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_index16_predict.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2q_tests.log 2>&1; tail -n 3 gpurun_out/r2q_tests.log
L="1024,64,0,65600 1024,128,0,65600 512,64,0,65664 512,64,0,65600 256,64,0,65664 256,64,0,65600 1024,64,0,65664"
timeout 900 python tools/time_launches.py c5 ELL --index16 2 --reps 10 $L > gpurun_out/r2q_tl.log 2>&1
timeout 900 python tools/time_launches.py c5 ELL --index16 0 --reps 10 256,64,0,65664 1024,64,0,65600 512,64,0,65664 >> gpurun_out/r2q_tl.log 2>&1
timeout 600 python tools/time_launches.py c2 ELL --index16 2 --reps 50 1024,64,0,65600 128,64,25,65600 256,64,0,65600 >> gpurun_out/r2q_tl.log 2>&1
cat gpurun_out/r2q_tl.log
timeout 600 python tools/power_probe.py c5 ELL 2 --launch 1024,64,0,65600 > gpurun_out/r2q_probe.log 2>&1; cat gpurun_out/r2q_probe.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dict_flags|k_ell_fill" -c 2 --csv python tools/kernel_one.py c5 ELL 1 --index16 2 --launch 1024,64,0,65600 2>&1 | grep -E "k_dict|k_ell_fill" | cut -d, -f5,15
( time timeout 1800 python bench.py ) > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2q_bench.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ['value','ms_per_step','step_phases_ms','steps_ms','clocks','e2e','mflops_per_w','gpu_launches']}); print(d['config']); print(d['roofline'])
print({c: (v.get('format'), v.get('kernel_us'), v.get('frac_measured_peak'), v.get('frac_gather_ceiling'), v.get('leg_seconds')) for c, v in d.get('per_config', {}).items()})"
tail -n 3 gpurun_out/r2q_bench.err
