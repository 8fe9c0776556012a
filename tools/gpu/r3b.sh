#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "nnz_split" > gpurun_out/r3b_new.log 2>&1; tail -n 2 gpurun_out/r3b_new.log
T=gpurun_out/r3b_tl.log
L=""
for b in 64 128 256; do for r in 32 64; do for k in 0x404 0x408; do L="$L $b,$r,-1,$k"; done; done; done
timeout 600 python tools/time_launches.py c3 CSR --csr-alg 3 --reps 10 $L > $T 2>&1
timeout 600 python tools/time_launches.py c4 CSR --csr-alg 3 --reps 10 $L >> $T 2>&1
cat $T
timeout 1200 python bench.py > gpurun_out/r3b_bench.json 2> gpurun_out/r3b_bench.err; tail -n 3 gpurun_out/r3b_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r3b_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['steps_ms'], d['roofline']['frac'], d['clocks'], d['config']['pool_priming_steps_ms'])
for s in d['steps_phase_ms']['per_step']: print(s)"
