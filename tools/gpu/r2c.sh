#!/bin/bash
# r2 session C: tile-kernel parity, sweep of COO/HYB/merge with tile knobs, ncu traffic per label, c5 bench (slab launch tune)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "tile or launch_variants or determinism" > gpurun_out/r2c_parity.log 2>&1
tail -3 gpurun_out/r2c_parity.log
timeout 1500 python tools/format_sweep.py --configs c2,c3,c4 --formats CSR-merge,HYB,COO --out gpurun_out/r2c_fs > gpurun_out/r2c_fs.log 2>&1
tail -12 gpurun_out/r2c_fs.log
timeout 900 python tools/ncu_traffic.py c5 ELL --launch "ELL=256,64,0,65664" > gpurun_out/r2c_ncu_c5.log 2>&1
timeout 1500 python tools/ncu_traffic.py c2 ELL-16 SELL-16 ELL SELL CSR-stream COO CSR-vector CSR-merge > gpurun_out/r2c_ncu_c2.log 2>&1
timeout 1500 python tools/ncu_traffic.py c3 COO HYB CSR-merge > gpurun_out/r2c_ncu_c3.log 2>&1
timeout 1500 python tools/ncu_traffic.py c4 ELL SELL CSR-vector COO > gpurun_out/r2c_ncu_c4.log 2>&1
cp profiles/ncu_traffic_c*.json gpurun_out/ 2>/dev/null
( time timeout 1200 python bench.py --per-config none --no-cpu-baseline ) > gpurun_out/r2c_bench_c5.json 2> gpurun_out/r2c_bench_c5.err
tail -c 1200 gpurun_out/r2c_bench_c5.json; tail -4 gpurun_out/r2c_bench_c5.err
cat gpurun_out/r2c_ncu_c*.log | cut -c 1-400
