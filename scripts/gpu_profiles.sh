#!/bin/bash
# refresh the committed evidence: launch list, ncu full captures, sanitizers
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 6 --warmup 2 --ttt 0 --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reg2d -s 3 -c 1 -o gpurun_out/prof_reg2d -f python bench.py --steps 4 --warmup 2 --ttt 0 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:classic2d -s 3 -c 1 -o gpurun_out/prof_classic2d -f python bench.py --mode classic --steps 4 --warmup 2 --ttt 0 --no-cpu > gpurun_out/ncu_full_classic.log 2>&1; echo "ncu classic rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
