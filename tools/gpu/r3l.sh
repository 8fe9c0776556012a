#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_index16_predict.py tests/test_gpu_parity.py -x -q -k "index16 or dict or 8 or layouts" > gpurun_out/r3l_tests.log 2>&1; tail -n 2 gpurun_out/r3l_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dict_flags|k_ell_fill" -c 2 --csv python tools/kernel_one.py c5 ELL 1 --index16 2 --launch 1024,64,0,64 > gpurun_out/r3l_ncu.csv 2>&1; grep -E "k_dict|k_ell_fill" gpurun_out/r3l_ncu.csv | cut -d, -f5,15 | cut -c1-140
timeout 900 python bench.py --per-config none --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/r3l_bench.json 2> gpurun_out/r3l_bench.err; tail -n 2 gpurun_out/r3l_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r3l_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['steps_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['step_phases_ms'])"
