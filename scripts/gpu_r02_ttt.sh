#!/bin/bash
# round 2: compute-sanitizer over every kernel family, the bench + launch list + ncu capture of the
# cycle kernel (round-2 evidence), then the MEASURED time-to-1e-6 on 16384^2 (hours; segments logged to
# gpurun_out/ttt_1e-06_16384.jsonl as they finish)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash scripts/gpu_sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1; cat gpurun_out/sanitize_summary.txt
timeout 900 python bench.py > gpurun_out/bench_r02.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r02.log; tail -2 gpurun_out/bench_r02.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 6 --warmup 2 --ttt 0 --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reg2d -s 3 -c 1 -o gpurun_out/prof_reg2d_r02 -f python bench.py --steps 4 --warmup 2 --ttt 0 --no-cpu --no-mg > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 60000 > gpurun_out/ttt_clocks.csv 2>/dev/null &
SMI=$!
timeout ${TTT_LIMIT:-19000} python scripts/ttt_1e6.py > gpurun_out/ttt.log 2>&1; echo "ttt rc=$?" >> gpurun_out/ttt.log
kill $SMI 2>/dev/null
tail -3 gpurun_out/ttt.log
