#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
( for v in 0 1; do HJ_REG2D_VARIANT=$v timeout 300 python scripts/kt.py "k=16" "k=1" "k=4" "k=64"; done
  timeout 300 python scripts/kt.py "mode=classic" "dtype=f32,k=16" "kernel=smem,k=16" ) 2>&1 | tee gpurun_out/kt.log
