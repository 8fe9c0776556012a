#!/bin/bash
# r2 session A: gather ceiling, per-format sweep with L2 policies, parity, c3 ncu traffic
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2a_smi.txt
timeout 300 python tools/gather_ceiling.py c3 c4 --json gpurun_out/r2a_gather.json > gpurun_out/r2a_gather.log 2>&1
timeout 900 python tools/format_sweep.py --configs c2,c3,c4 --formats CSR-vector,CSR-merge,CSR-stream,ELL,ELL-16,SELL,SELL-16,HYB,COO --out gpurun_out/r2a_fs > gpurun_out/r2a_fs.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2a_parity.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__throughput.avg.pct_of_peak_sustained_elapsed
timeout 300 ncu --metrics $M --clock-control none -k regex:k_coo -c 2 --csv python tools/kernel_one.py c3 COO 3 > gpurun_out/r2a_ncu_c3_coo.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:k_csr_merge -c 2 --csv python tools/kernel_one.py c3 CSR 3 --csr-alg 3 > gpurun_out/r2a_ncu_c3_merge.csv 2>&1
tail -3 gpurun_out/r2a_parity.log
cat gpurun_out/r2a_gather.log
tail -40 gpurun_out/r2a_fs.log
