for i in 1 2; do
GBM3D_LIB=paper_2103_10765_b200/libgbm3d.so python tools/dev/time_host.py c4
GBM3D_LIB=variants/host16.so python tools/dev/time_host.py c4
GBM3D_LIB=paper_2103_10765_b200/libgbm3d.so python tools/dev/time_host.py c3
GBM3D_LIB=variants/host16.so python tools/dev/time_host.py c3
done
