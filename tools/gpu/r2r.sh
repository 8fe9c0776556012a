#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
A="--per-config none --no-cpu-baseline --no-e2e --steps 8"
for v in a b c; do
  case $v in
    a) E="" ; W=3 ;;
    b) E="BENCH_NO_POWER_SAMPLES=1 BENCH_NO_CLOCKS=1"; W=3 ;;
    c) E=""; W=6 ;;
  esac
  env $E timeout 900 python bench.py $A --warmup $W > gpurun_out/r2r_$v.json 2> gpurun_out/r2r_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2r_$v.json').read().strip().splitlines()[-1])
print('$v', d['value'], d['steps_ms'], d['clocks']); print(d['steps_phase_ms'])"
done
