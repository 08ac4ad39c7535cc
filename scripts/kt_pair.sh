#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
HJ_REG2D_VARIANT=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_overlap.py -m gpu -q -x -k "hier2d or counts or overlap or 16384 or determinism" > gpurun_out/pytest_pair.log 2>&1; tail -3 gpurun_out/pytest_pair.log
( for v in 0 3; do HJ_REG2D_VARIANT=$v timeout 300 python scripts/kt.py "k=16" "k=64" "k=4" "dtype=f32,k=16" "dtype=f32,k=64"; done ) 2>&1 | tee gpurun_out/kt_pair.log
