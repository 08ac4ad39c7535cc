#!/bin/bash
# usage: gpu_check.sh [tests] [bench] [ncu] [launches]   (runs on the gpurun box)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests) timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log;;
    quick) timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -x -k "not 16384 and not config3" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log; tail -3 gpurun_out/pytest_quick.log;;
    bench) timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; tail -2 gpurun_out/bench.log | cut -c1-600;;
    benchfast) timeout 600 python bench.py --ttt 0 --no-cpu > gpurun_out/benchfast.log 2>&1; tail -2 gpurun_out/benchfast.log | cut -c1-400;;
    launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 6 --warmup 2 --ttt 0 --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?";;
    ncu) timeout 900 ncu --set full --clock-control none --import-source on -k regex:reg2d -s 3 -c 1 -o gpurun_out/prof_reg2d -f python bench.py --steps 4 --warmup 2 --ttt 0 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log;;
  esac
done
