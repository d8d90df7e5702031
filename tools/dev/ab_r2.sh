#!/bin/bash
# dev: new build vs round-1 build on c3/c4 timing, then the matcher parity tests
mkdir -p gpurun_out
for lib in paper_2103_10765_b200/libgbm3d.so; do
  for c in c3 c4; do
    GBM3D_LIB=$lib timeout 120 python tools/time_config.py --config $c --reps 10 2>&1 | tail -1 | sed "s|^|$lib |"
  done
done
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
