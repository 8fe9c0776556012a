#!/bin/bash
# Session-3 verification: full GPU suite, smoke, c5 headline ncu traffic at the bench launch, launch list of a
# timed bench step, DRAM bytes of the gather-only kernel on c3 (x re-read without matrix stream / y / records).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/r3g_tests.log 2>&1; tail -n 3 gpurun_out/r3g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3g_smoke.log 2>&1; tail -n 1 gpurun_out/r3g_smoke.log
timeout 900 python tools/ncu_traffic.py c5 ELL-8 --launch "ELL-8=1024,64,0,64" --out gpurun_out/r3g_ncu_traffic_c5.json > gpurun_out/r3g_traffic.log 2>&1; tail -n 5 gpurun_out/r3g_traffic.log
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" --csv --log-file gpurun_out/r3g_launches.csv python bench.py --steps 1 --warmup 1 --prime 0 --per-config none --no-cpu-baseline --no-e2e > gpurun_out/r3g_ncu_bench.log 2>&1
tail -n 2 gpurun_out/r3g_ncu_bench.log; wc -l gpurun_out/r3g_launches.csv
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gather --csv python tools/gather_ceiling.py c3 --reps 1 > gpurun_out/r3g_gather_dram.csv 2>&1; grep -E "gather|dram" gpurun_out/r3g_gather_dram.csv | head -20
