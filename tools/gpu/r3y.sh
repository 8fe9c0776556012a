#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPMV_ELL_FILL_WARP=1 timeout 1200 python -m pytest tests/test_gpu_index16_predict.py tests/test_gpu_parity.py -x -q -k "index16 or dict or 8 or layouts" > gpurun_out/r3y_tests.log 2>&1; tail -n 2 gpurun_out/r3y_tests.log
for w in 0 1; do
  if [ $w = 1 ]; then export SPMV_ELL_FILL_WARP=1; else unset SPMV_ELL_FILL_WARP; fi
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_ell_fill" -c 1 --csv python tools/kernel_one.py c5 ELL 1 --index16 2 --launch 1024,64,0,64 > gpurun_out/r3y_ncu_$w.csv 2>&1
  echo "warp=$w"; grep -E "k_ell_fill" gpurun_out/r3y_ncu_$w.csv | awk -F'","' '{print $13, $15}'
done
