#!/bin/bash
# Before/after ncu of the merge-path family on c3 (tile walk 0x104 = round-2 best, row-map nnz-split 0x808) with COO.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sector_hit_rate.pct,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
for v in "CSR 128,32,50,260 3 mtile" "CSR 64,64,-1,2056 3 rowmap" "COO 64,64,0,8 0 coo"; do
  set -- $v
  timeout 600 ncu --metrics $M --clock-control none --profile-from-start off -k regex:"k_csr_merge|k_csr_nnz|k_coo" -c 1 --csv python tools/kernel_one.py c3 $1 1 --launch $2 --csr-alg $3 > gpurun_out/r3s_$4.csv 2>&1
  echo "== $4"; grep -E "k_csr|k_coo" gpurun_out/r3s_$4.csv | awk -F'","' '{print $13, $15}' | head -n 14
done
timeout 900 python tools/ncu_traffic.py c3 CSR-merge --launch "CSR-merge=64,64,-1,2056" --out gpurun_out/r3s_traffic_c3.json > gpurun_out/r3s_traffic.log 2>&1; tail -n 1 gpurun_out/r3s_traffic.log | cut -c1-400
