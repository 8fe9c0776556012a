#!/bin/bash
# r2 session E: host-phase breakdown of the c5 step (ELL-8), index8 + merge-stream parity, merge sweep on c3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 900 python bench.py --per-config none --no-cpu-baseline --no-e2e --steps 5 ) > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2e_bench.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ['value','ms_per_step','step_phases_ms','host_phases_ms','host_ms_per_step','clocks']}); print(d['config']['format'], d['config']['launch'], d['roofline']['kernel_avg_us'], d['roofline']['frac'])"
tail -3 gpurun_out/r2e_bench.err
timeout 1500 python -m pytest tests/test_gpu_index16_predict.py tests/test_gpu_parity.py -x -q > gpurun_out/r2e_tests.log 2>&1; tail -3 gpurun_out/r2e_tests.log
timeout 900 python tools/format_sweep.py --configs c3,c2 --formats CSR-merge --out gpurun_out/r2e_fs > gpurun_out/r2e_fs.log 2>&1; tail -4 gpurun_out/r2e_fs.log
timeout 600 python tools/time_launches.py c3 CSR --csr-alg 3 128,255,-1,0x204 128,255,-1,0x208 256,255,-1,0x204 256,255,-1,0x208 256,128,-1,0x210 512,64,-1,0x204 512,64,-1,0x208 128,32,50,0x104 > gpurun_out/r2e_tl.log 2>&1; cat gpurun_out/r2e_tl.log
