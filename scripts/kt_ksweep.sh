#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
( HJ_REG2D_VARIANT=2 timeout 300 python scripts/kt.py "k=16" "k=64"
  timeout 600 python scripts/kt.py "k=1" "k=2" "k=4" "k=8" "k=16" "k=32" "k=64" "mode=classic" "dtype=f32,k=16" "dtype=f32,k=4" "dtype=f32,k=64" "dtype=f32,mode=classic" ) 2>&1 | tee gpurun_out/kt_ksweep.log
