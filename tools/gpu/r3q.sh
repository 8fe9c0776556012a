#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
A="--per-config none --no-cpu-baseline --steps 4"
for v in a b c; do
  case $v in
    a) E="BENCH_DEBUG_MEM=1" ;;
    b) E="BENCH_DEBUG_MEM=1 BENCH_E2E_TRIM=1" ;;
    c) E="BENCH_DEBUG_MEM=1 BENCH_E2E_RELEASE_INPUT=1 BENCH_E2E_RELEASE_CSR=1 BENCH_E2E_DEPTH=2 BENCH_E2E_TRIM=1" ;;
  esac
  env $E timeout 1200 python bench.py $A > gpurun_out/r3q_$v.json 2> gpurun_out/r3q_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/r3q_$v.json').read().strip().splitlines()[-1])
print('$v', d['value'], d['e2e'])" 2>&1 | tail -n 1
  grep "\[e2e\]" gpurun_out/r3q_$v.err | tail -n 12
done
