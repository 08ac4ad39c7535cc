#!/bin/bash
# multigrid kernels: ncu --set full of the fine restriction and the fused post-smoothing cycle,
# sanitizer runs over every kernel family, smoke
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mg_restrict2d -c 1 -o gpurun_out/prof_mg_restrict -f python scripts/mg_launches.py > gpurun_out/ncu_mg_restrict.log 2>&1; echo "ncu restrict rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:Li2ELb1E -s 8 -c 1 -o gpurun_out/prof_mg_post -f python scripts/mg_launches.py > gpurun_out/ncu_mg_post.log 2>&1; echo "ncu post rc=$?"
