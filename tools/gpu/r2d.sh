#!/bin/bash
# r2 session D: 8-bit dictionary ELL/SELL — parity, sweep, default bench, ncu traffic of the bench kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; tail -2 gpurun_out/r2d_smoke.log
timeout 1500 python -m pytest tests/test_gpu_index16_predict.py tests/test_gpu_parity.py -x -q > gpurun_out/r2d_tests.log 2>&1; tail -3 gpurun_out/r2d_tests.log
timeout 900 python tools/format_sweep.py --configs c2 --formats ELL,ELL-16,ELL-8,SELL,SELL-16,SELL-8 --out gpurun_out/r2d_fs > gpurun_out/r2d_fs.log 2>&1; tail -8 gpurun_out/r2d_fs.log
( time timeout 1500 python bench.py ) > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
tail -c 2500 gpurun_out/r2d_bench.json; tail -4 gpurun_out/r2d_bench.err
L=$(python -c "import json; d=json.loads(open('gpurun_out/r2d_bench.json').read().strip().splitlines()[-1]); c=d['config']; l=c['launch']; print(c['format']+'='+','.join(str(l[k]) for k in ('block','maxreg','carveout_pct','knob')))")
LAB=${L%%=*}
timeout 900 python tools/ncu_traffic.py c5 $LAB --launch "$L" > gpurun_out/r2d_ncu_c5.log 2>&1
timeout 900 python tools/ncu_traffic.py c2 ELL-8 SELL-8 > gpurun_out/r2d_ncu_c2.log 2>&1
cp profiles/ncu_traffic_c*.json gpurun_out/ 2>/dev/null
cat gpurun_out/r2d_ncu_c*.log | cut -c 1-600
