#!/bin/bash
# One gpurun session: GPU tests, bench, launch list, ncu full capture of the top kernel.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-also --cpu-seconds 1 > gpurun_out/bench_small.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-also --cpu-seconds 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 120 python tools/run_once.py --config c3 > gpurun_out/plain_c3.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -c 2 \
   -o gpurun_out/prof_c3 python tools/run_once.py --config c3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
