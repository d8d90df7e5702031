#!/bin/bash
# dev: end-to-end host-buffer timing per variant library (c3, c4)
for lib in variants/lib_*.so; do for c in c3 c4; do GBM3D_LIB=$lib timeout 120 python tools/dev/time_host.py $c 2>&1 | tail -1 | sed "s|^|$lib |"; done; done
