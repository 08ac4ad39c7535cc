#!/bin/bash
# full pass: gpu tests, bench, launch list, ncu full capture of the cycle kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; tail -2 gpurun_out/bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 6 --warmup 2 --ttt 0 --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reg2d -s 3 -c 1 -o gpurun_out/prof_reg2d -f python bench.py --steps 4 --warmup 2 --ttt 0 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:classic2d -s 3 -c 1 -o gpurun_out/prof_classic2d -f python bench.py --mode classic --steps 4 --warmup 2 --ttt 0 --no-cpu > gpurun_out/ncu_full_classic.log 2>&1; echo "ncu classic rc=$?"
