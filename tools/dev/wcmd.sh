mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:s1_syn_xy --launch-skip 2 -c 1 -o gpurun_out/s1_syn1 -f python tools/dev/stage1_once.py c3 > gpurun_out/ncu_s1c.log 2>&1; tail -1 gpurun_out/ncu_s1c.log
