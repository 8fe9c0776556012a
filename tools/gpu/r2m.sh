#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python tools/overhead_corpus.py --out gpurun_out/overhead_corpus.jsonl > gpurun_out/r2m.log 2>&1
tail -n 5 gpurun_out/r2m.log; wc -l gpurun_out/overhead_corpus.jsonl
