#!/bin/bash
# The c5 headline's launch variants inside the sustained power loop (the offline refine times short bursts).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
A="--per-config none --no-cpu-baseline --no-e2e --steps 4 --format ELL"
for L in 1024,64,0,64 1024,255,0,64 512,64,0,64 1024,64,0,65600 1024,255,0,65600 512,64,0,65664; do
  timeout 900 python bench.py $A --launch $L > gpurun_out/r4j.json 2> gpurun_out/r4j.err
  python -c "
import json;d=json.loads(open('gpurun_out/r4j.json').read().strip().splitlines()[-1])
print('$L', d['value'], d['roofline']['kernel_avg_us'], d['clocks']['sm_mhz'], d['config']['format'])" 2>&1 | tail -n 1
done
