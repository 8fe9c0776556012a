#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_index16_predict.py tests/test_gpu_parity.py -x -q -k "index16 or dict or 8 or layouts" > gpurun_out/r3m_tests.log 2>&1; tail -n 2 gpurun_out/r3m_tests.log
for b in 3 2 4 6 32; do
  SPMV_ELL_FILL_BPS=$b timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dict_flags|k_ell_fill" -c 2 --csv python tools/kernel_one.py c5 ELL 1 --index16 2 --launch 1024,64,0,64 > gpurun_out/r3m_ncu_$b.csv 2>&1
  echo "bps=$b"; grep -E "k_dict|k_ell_fill" gpurun_out/r3m_ncu_$b.csv | awk -F'","' '{print substr($5,1,40), $(NF)}'
done
