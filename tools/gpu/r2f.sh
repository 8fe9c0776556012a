#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 900 python bench.py --per-config none --no-cpu-baseline --no-e2e --steps 6 ) > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2f_bench.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ['value','ms_per_step','step_phases_ms','host_phases_ms','steps_ms','device_gaps_ms','host_ms_per_step','clocks']}); print(d['config']['format'], d['config']['launch'], d['roofline']['kernel_avg_us'], d['roofline']['frac'])"
tail -3 gpurun_out/r2f_bench.err
timeout 600 python tools/time_launches.py c2 COO 128,255,-1,8 128,255,-1,0x104 256,255,-1,0x104 256,255,-1,0x108 512,64,-1,0x104 512,64,-1,0x108 1024,64,-1,0x104 > gpurun_out/r2f_tl.log 2>&1; cat gpurun_out/r2f_tl.log
timeout 600 python tools/time_launches.py c2 CSR --csr-alg 3 128,255,-1,0x204 128,255,-1,0x208 256,255,-1,0x204 256,255,-1,0x208 256,128,-1,0x210 512,64,-1,0x204 512,64,-1,0x208 >> gpurun_out/r2f_tl.log 2>&1; tail -7 gpurun_out/r2f_tl.log
