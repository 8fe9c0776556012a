#!/bin/bash
# Best-suited-matrix sweep: every format, launch-tuned, on the three extra large matrices.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python tools/format_sweep.py --configs lap2d_4096,band64_2M,lap2d_long_4096 --out gpurun_out/r2x_best_suited > gpurun_out/r2x.log 2>&1
tail -n 50 gpurun_out/r2x.log
