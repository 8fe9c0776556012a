#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
A="--per-config none --no-cpu-baseline --no-e2e --steps 6"
for v in a b c; do
  case $v in
    a) E="BENCH_DEBUG_MEM=1" ;;
    b) E="BENCH_DEBUG_MEM=1 BENCH_NO_KEVENTS=1" ;;
    c) E="BENCH_DEBUG_MEM=1 BENCH_NO_CLOCKS=1 BENCH_NO_POWER_SAMPLES=1" ;;
  esac
  env $E timeout 900 python bench.py $A > gpurun_out/r3c_$v.json 2> gpurun_out/r3c_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/r3c_$v.json').read().strip().splitlines()[-1])
print('$v', d['value'], d['steps_ms'], d['config']['pool_priming_steps_ms'])
for s in d['steps_phase_ms']['per_step']: print(s)"
  grep "\[mem\]" gpurun_out/r3c_$v.err | tail -n 14
done
