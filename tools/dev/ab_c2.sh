#!/bin/bash
# dev: c2 timing per variant library and strip split count, c2 parity of each library
for pass in 1; do
for lib in variants/lib_*.so; do
  for sp in 0 1 2 3 4; do
    GBM3D_STRIP_SPLIT=$sp GBM3D_LIB=$lib timeout 60 python tools/time_config.py --config c2 --reps 20 2>&1 | tail -1 | sed "s|^|$lib split=$sp |"
  done
done
done
for lib in variants/lib_*.so; do GBM3D_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c2 or fuzz" 2>&1 | tail -1 | sed "s|^|$lib |"; done
