#!/bin/bash
# Bench + launch list + ncu full captures (c3, c4) of the current build.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-also --step-only > gpurun_out/bench_small.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-also --step-only > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-also --cpu-seconds 1 > gpurun_out/bench_small_all.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
   --log-file gpurun_out/launches_all.csv python bench.py --steps 3 --warmup 3 --no-also --cpu-seconds 1 > gpurun_out/ncu_launch_all.log 2>&1; echo "ncu launches (all legs) rc=$?"
timeout 120 python tools/run_once.py --config c3 > gpurun_out/plain_c3.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc16 -c 1 \
   -o gpurun_out/prof_c3 python tools/run_once.py --config c3 > gpurun_out/ncu_full.log 2>&1; echo "ncu c3 rc=$?"
timeout 120 python tools/run_once.py --config c4 > gpurun_out/plain_c4.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc16 -c 1 \
   -o gpurun_out/prof_c4 python tools/run_once.py --config c4 > gpurun_out/ncu_full4.log 2>&1; echo "ncu c4 rc=$?"
