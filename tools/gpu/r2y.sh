#!/bin/bash
# c3: merge-path variants vs COO, live timings + one ncu --set full capture each.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/time_launches.py c3 CSR --csr-alg 3 --reps 20 64,64,0,4 64,64,0,8 64,128,0,8 128,64,0,16 128,32,50,260 128,64,0,264 256,128,-1,528 128,128,-1,516 > gpurun_out/r2y_tl.log 2>&1
cat gpurun_out/r2y_tl.log
for v in "CSR 64,64,0,8 3 merge8" "CSR 128,32,50,260 3 mtile4" "COO 64,64,0,8 0 coo8"; do
  set -- $v
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_csr_merge|k_coo" -c 1 -o gpurun_out/r2y_$4 python tools/kernel_one.py c3 $1 1 --launch $2 --csr-alg $3 > gpurun_out/r2y_$4.log 2>&1
  tail -n 1 gpurun_out/r2y_$4.log
done
