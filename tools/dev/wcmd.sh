for v in main; do lib=paper_2103_10765_b200/libgbm3d.so; echo $v; GBM3D_LIB=$lib python tools/dev/time_host.py c3; GBM3D_LIB=$lib python tools/dev/time_host.py c4; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host or row_ranges or batched" 2>&1 | tail -2
