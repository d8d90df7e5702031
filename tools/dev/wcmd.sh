for rep in 1 2; do
for v in main sleep_20 sleep_64 sleep_128; do lib=variants/$v.so; [ $v = main ] && lib=paper_2103_10765_b200/libgbm3d.so; echo -n "$v "; GBM3D_LIB=$lib python tools/time_config.py --config c3 --reps 20; echo -n "$v "; GBM3D_LIB=$lib python tools/time_config.py --config c4 --reps 10; done
done
