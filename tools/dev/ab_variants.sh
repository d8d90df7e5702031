#!/bin/bash
# dev: time c3/c4 for every variants/lib_*.so (two passes, interleaved), plus c0 parity per lib
for pass in 1 2; do
for lib in variants/lib_*.so; do
  for c in c3 c4; do
    GBM3D_LIB=$lib timeout 30 python tools/time_config.py --config $c --reps 10 2>&1 | tail -1 | sed "s|^|$lib |"
  done
done
done
for lib in variants/lib_*.so; do GBM3D_LIB=$lib timeout 60 python tools/dev/one_c0.py 2>&1 | tail -1 | sed "s|^|$lib |"; done
