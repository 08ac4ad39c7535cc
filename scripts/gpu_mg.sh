#!/bin/bash
# multigrid: GPU parity tests + ncu launch list of 2 V-cycles at 16383^2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_mg.py -x -q > gpurun_out/pytest_mg.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_mg.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/mg_launches.csv python scripts/mg_launches.py > gpurun_out/mg_launches.log 2>&1; echo "ncu rc=$?"
