mkdir -p gpurun_out
for v in w_v4 w_v10 w_v11 w_v4 w_v10 w_v11; do echo $v; GBM3D_LIB=variants/$v.so python tools/dev/time_wiener.py c3; done
GBM3D_LIB=variants/w_v11.so timeout 900 python -m pytest tests/test_gpu_wiener.py tests/test_gpu_denoise.py -q -x 2>&1 | tail -2
