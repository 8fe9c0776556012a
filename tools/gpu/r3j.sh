#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize_cases.py ragged_empty,long_rows,rmat10,mixed_tiles > gpurun_out/r3j_$t.log 2>&1
  echo "== $t"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^ok" gpurun_out/r3j_$t.log | tail -n 8
done
