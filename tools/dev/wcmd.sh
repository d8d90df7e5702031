mkdir -p gpurun_out
for v in s1_old s8_141 s8_181 s8_282 main; do
  lib=variants/$v.so; [ $v = main ] && lib=paper_2103_10765_b200/libgbm3d.so
  GBM3D_LIB=$lib TAG=$v python tools/dev/time_match.py c3 8 8 19 16
done
GBM3D_LIB=paper_2103_10765_b200/libgbm3d.so TAG=r16 python tools/dev/time_match.py c3 8 8 16 16
GBM3D_LIB=variants/s1_old.so TAG=r16old python tools/dev/time_match.py c3 8 8 16 16
python -c "
import numpy as np
for t in ['s8_141','s8_181','s8_282','main']:
    print(t, all((np.load(f'gpurun_out/m_{t}_{a}.npy')==np.load(f'gpurun_out/m_s1_old_{a}.npy')).all() for a in ('idx','dist')))
print('r16', all((np.load(f'gpurun_out/m_r16_{a}.npy')==np.load(f'gpurun_out/m_r16old_{a}.npy')).all() for a in ('idx','dist')))
"
