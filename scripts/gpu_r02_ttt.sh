#!/bin/bash
# round 2: compute-sanitizer over every kernel family (after the last kernel change), then the MEASURED
# time-to-1e-6 on 16384^2 (hours; segments logged to gpurun_out/ttt_1e-06_16384.jsonl as they finish)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash scripts/gpu_sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1; cat gpurun_out/sanitize_summary.txt
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 60000 > gpurun_out/ttt_clocks.csv 2>/dev/null &
SMI=$!
timeout ${TTT_LIMIT:-19800} python scripts/ttt_1e6.py > gpurun_out/ttt.log 2>&1; echo "ttt rc=$?" >> gpurun_out/ttt.log
kill $SMI 2>/dev/null
tail -3 gpurun_out/ttt.log
