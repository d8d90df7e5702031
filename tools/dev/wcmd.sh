GBM3D_LIB=paper_2103_10765_b200/libgbm3d.so python tools/dev/time_small.py
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gather.py -q -x 2>&1 | tail -1
