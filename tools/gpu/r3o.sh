#!/bin/bash
# The N > 1 branch of the bench at the c5 size: 2 and 4 virtual ranks (in-process communicator group) on one GPU.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for W in 2 4; do
  timeout 1500 python bench.py --gpus $W --virtual --config c5 --steps 3 --warmup 3 --per-config none --no-cpu-baseline > gpurun_out/r3o_v$W.json 2> gpurun_out/r3o_v$W.err; tail -n 2 gpurun_out/r3o_v$W.err
  python -c "
import json;d=json.loads(open('gpurun_out/r3o_v$W.json').read().strip().splitlines()[-1])
print($W, d['value'], d['scaling'], d['config']['plan'], d['roofline']['frac'], d['config']['format'], d.get('lambda_last'))"
done
