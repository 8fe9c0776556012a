#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "create or ingest or csr_bit or unsorted or errors or fullsize" > gpurun_out/r3w_tests.log 2>&1; tail -n 2 gpurun_out/r3w_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests.sum --clock-control none -k regex:"k_check" -c 1 --csv python tools/kernel_one.py c5 ELL 1 --index16 2 --launch 1024,64,0,64 > gpurun_out/r3w_ncu.csv 2>&1; grep -E "k_check" gpurun_out/r3w_ncu.csv | awk -F'","' '{print $13, $15}'
timeout 900 python bench.py --per-config none --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/r3w_bench.json 2> gpurun_out/r3w_bench.err; tail -n 2 gpurun_out/r3w_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r3w_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['steps_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['step_phases_ms'])"
