#!/bin/bash
# Round-2 measurement run: bench line, launch list of the timed step, ncu --set full of the
# matcher (c3, c4), and the integer-peak microkernels' SASS pipes.  Results in gpurun_out/;
# tools/make_ncu_counters.py turns the captures into profiles/ncu_counters.json.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import paper_2103_10765_b200 as g; print(g.version())" > gpurun_out/build_id.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-also --step-only > gpurun_out/bench_small.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-also --step-only > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 120 python tools/run_once.py --config c3 > gpurun_out/plain_c3.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_tc16 -c 1 \
   -o gpurun_out/prof_c3 -f python tools/run_once.py --config c3 > gpurun_out/ncu_full.log 2>&1; echo "ncu c3 rc=$?"
timeout 120 python tools/run_once.py --config c4 > gpurun_out/plain_c4.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_tc16 -c 1 \
   -o gpurun_out/prof_c4 -f python tools/run_once.py --config c4 > gpurun_out/ncu_full4.log 2>&1; echo "ncu c4 rc=$?"
timeout 120 python tools/run_once.py --config c2 > gpurun_out/plain_c2.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_tcp -c 1 \
   -o gpurun_out/prof_c2 -f python tools/run_once.py --config c2 > gpurun_out/ncu_full2.log 2>&1; echo "ncu c2 rc=$?"
