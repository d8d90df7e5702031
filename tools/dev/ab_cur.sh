#!/bin/bash
# dev: c0 parity of every variant, matcher parity tests (on $PARITY_LIB, default the in-tree
# build), then c3/c4 timing of every variant
for lib in variants/lib_*.so; do GBM3D_LIB=$lib timeout 60 python tools/dev/one_c0.py 2>&1 | tail -1 | sed "s|^|$lib |"; done
GBM3D_LIB=${PARITY_LIB:-paper_2103_10765_b200/libgbm3d.so} timeout 400 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 900 bash tools/dev/ab_variants.sh 2>&1 | grep -v "idx True"
