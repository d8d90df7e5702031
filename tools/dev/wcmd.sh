for i in 1 2; do for v in main ana5; do lib=variants/$v.so; [ $v = main ] && lib=paper_2103_10765_b200/libgbm3d.so; echo -n "$v "; GBM3D_LIB=$lib TAG=$v python tools/dev/time_stage1.py c3; done; done
GBM3D_LIB=variants/ana5.so timeout 600 python -m pytest tests/test_gpu_stage1.py -q -x 2>&1 | tail -1
