#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
( for s in 0 300 700 1200 2000; do echo "stagger=$s"; HJ_STAGGER_NS=$s timeout 300 python scripts/kt.py "k=16" "k=64"; done ) 2>&1 | tee gpurun_out/kt_stagger.log
