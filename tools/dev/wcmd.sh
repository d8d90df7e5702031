for v in g_1024_5120 g_1024_4608 g_1024_4096 g_512_3072; do lib=variants/$v.so; echo $v; GBM3D_LIB=$lib python tools/dev/time_gather.py c3; GBM3D_LIB=$lib python tools/dev/time_gather.py c4; done
