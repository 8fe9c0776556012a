#!/bin/bash
# nnz-split CSR (merge family): parity + timings; bench with the pool-size rounding.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "nnz_split or launch_variants or determinism" > gpurun_out/r3a_new.log 2>&1; tail -n 3 gpurun_out/r3a_new.log
T=gpurun_out/r3a_tl.log
L=""
for b in 64 128 256 512; do for r in 32 64 128; do for k in 0x404 0x408; do L="$L $b,$r,-1,$k"; done; done; done
timeout 600 python tools/time_launches.py c3 CSR --csr-alg 3 --reps 10 128,32,50,260 $L > $T 2>&1
timeout 600 python tools/time_launches.py c3 COO --reps 10 64,64,0,8 64,128,0,8 >> $T 2>&1
timeout 600 python tools/time_launches.py c2 CSR --csr-alg 3 --reps 20 128,128,100,528 $L >> $T 2>&1
timeout 600 python tools/time_launches.py c4 CSR --csr-alg 3 --reps 10 64,255,50,8 $L >> $T 2>&1
cat $T
timeout 1200 python bench.py > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err; tail -n 3 gpurun_out/r3a_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r3a_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['steps_ms'], d['roofline']['frac'], d['clocks'])
for s in d['steps_phase_ms']['per_step']: print(s)"
