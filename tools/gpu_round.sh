#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full capture of the top kernel.
set -x
CFG=${CFG:-c2}
TAG=${TAG:-r1}
python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
python bench.py --config $CFG > gpurun_out/bench_${CFG}_${TAG}.json 2> gpurun_out/bench_${CFG}_${TAG}.err
tail -c 600 gpurun_out/bench_${CFG}_${TAG}.json
FMT=$(python -c "import json; d=json.load(open('gpurun_out/bench_${CFG}_${TAG}.json')); print(d['config']['format'])")
L=$(python -c "import json; d=json.load(open('gpurun_out/bench_${CFG}_${TAG}.json'))['config']['launch']; print(f\"{d['block']},{d['maxreg']},{d['carveout_pct']},{d['knob']}\")")
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv \
  python bench.py --config $CFG --format $FMT --launch $L --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_sliced} -s 20 -c 2 -o gpurun_out/prof_${CFG}_${TAG} \
  python bench.py --config $CFG --format $FMT --launch $L --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${CFG}_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${CFG}_${TAG}.log
