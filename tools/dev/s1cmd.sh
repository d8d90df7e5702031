mkdir -p gpurun_out
GBM3D_LIB=variants/s1_old.so TAG=old python tools/dev/time_stage1.py c3
TAG=new python tools/dev/time_stage1.py c3
python -c "
import numpy as np; a=np.load('gpurun_out/s1_old.npy'); b=np.load('gpurun_out/s1_new.npy'); d=np.abs(a-b); print('old vs new: max', d.max(), 'mean', d.mean(), 'frac>1e-2', (d>1e-2).mean())"
timeout 1200 python -m pytest tests/test_gpu_stage1.py tests/test_gpu_denoise.py -q -x 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k "regex:s1_|gather_volume" --log-file gpurun_out/s1_launches3.csv python tools/dev/stage1_once.py c3 > gpurun_out/ncu_s1b.log 2>&1; tail -1 gpurun_out/ncu_s1b.log
