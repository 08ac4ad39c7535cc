#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
( for v in 0 2; do HJ_REG2D_VARIANT=$v timeout 300 python scripts/kt.py "k=16" "k=64" "dtype=f32,k=16"; done ) 2>&1 | tee gpurun_out/kt_var.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "hier2d or classic2d or counts" > gpurun_out/pytest_quick.log 2>&1; tail -2 gpurun_out/pytest_quick.log
