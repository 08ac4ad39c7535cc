#!/bin/bash
# one link of the time-to-1e-6 chain (resumes from the box's checkpoint when the lease lands on the same box)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 60000 > gpurun_out/ttt_clocks_$(date +%H%M%S).csv 2>/dev/null &
SMI=$!
TTT_WALL=${TTT_WALL:-2900} timeout 3450 python scripts/ttt_1e6.py > gpurun_out/ttt_$(date +%H%M%S).log 2>&1
kill $SMI 2>/dev/null
tail -2 gpurun_out/ttt_*.log | cut -c1-300
