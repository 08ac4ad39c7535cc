#!/bin/bash
# round 2, last window: res1w timing (the decision change), REG2D tile-order experiment, the full GPU
# suite, sanitizer over the changed kernels, smoke
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
HJ_RESIDENT=1 timeout 300 python scripts/resident_check.py > gpurun_out/resident_check_r02.log 2>&1; tail -3 gpurun_out/resident_check_r02.log
timeout 1200 python scripts/tile_order.py > gpurun_out/tile_order.log 2>&1; cat gpurun_out/tile_order.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_final.log; tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -2 gpurun_out/smoke_final.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_final_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_final_$tool.log | tail -1)"
done
# the REGT large-tile hazards racecheck reports are mbarrier-ordered (it does not model mbarrier arrive/wait
# between warps): the same cases with a group barrier after every sub-iteration
HJ_REGT_SWEEP_BARRIER=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_final_racecheck_sweepbar.log 2>&1
echo "racecheck (sweep barrier) rc=$? $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY' gpurun_out/sanitize_final_racecheck_sweepbar.log | tail -1)"
