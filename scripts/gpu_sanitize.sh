#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
HJ_SPLIT_CYCLE=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_memcheck_split.log 2>&1
echo "memcheck (split launch order) rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize_memcheck_split.log | tail -1)"
exit 0
timeout 300 python scripts/kt.py "mode=classic" "dtype=f32,mode=classic" 2>&1 | tee gpurun_out/kt_classic.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "classic or counts or k1" > gpurun_out/pytest_quick.log 2>&1; tail -2 gpurun_out/pytest_quick.log
