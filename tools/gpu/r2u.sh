#!/bin/bash
# COO on a TMA pipeline (knob 0x200|ept): parity, then timings vs the round-2 COO variants; then the full suite + bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coo_stream or determinism or launch_variants" > gpurun_out/r2u_new.log 2>&1; tail -n 3 gpurun_out/r2u_new.log
T=gpurun_out/r2u_tl.log
timeout 600 python tools/time_launches.py c2 COO --reps 50 128,64,0,8 128,128,-1,0x21a 128,255,-1,0x21a 128,128,-1,0x219 128,128,-1,0x220 64,128,-1,0x21a 64,255,-1,0x240 256,128,-1,0x210 256,128,-1,0x20d 512,64,-1,0x208 > $T 2>&1
timeout 600 python tools/time_launches.py c3 COO --reps 20 64,64,0,8 128,128,-1,0x210 128,128,-1,0x220 128,128,-1,0x20f 256,128,-1,0x210 256,128,-1,0x208 64,255,-1,0x240 >> $T 2>&1
timeout 600 python tools/time_launches.py c3 HYB --reps 20 64,64,25,8 128,128,-1,0x210 128,128,-1,0x220 256,128,-1,0x210 256,128,-1,0x208 64,255,-1,0x240 >> $T 2>&1
timeout 600 python tools/time_launches.py c4 COO --reps 20 64,32,0,4 128,128,-1,0x220 128,128,-1,0x21f 256,128,-1,0x210 64,255,-1,0x240 >> $T 2>&1
cat $T
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/r2u_tests.log 2>&1; tail -n 3 gpurun_out/r2u_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1; tail -n 2 gpurun_out/r2u_smoke.log
timeout 1200 python bench.py > gpurun_out/r2u_bench.json 2> gpurun_out/r2u_bench.err; tail -c 1500 gpurun_out/r2u_bench.json; tail -n 5 gpurun_out/r2u_bench.err
