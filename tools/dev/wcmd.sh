mkdir -p gpurun_out
timeout 600 python tools/dev/wiener_once.py c3 > gpurun_out/w_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wiener_tile -c 1 -o gpurun_out/prof_wiener_c3 -f python tools/dev/wiener_once.py c3 > gpurun_out/ncu_w.log 2>&1; echo "wiener ncu rc=$?"
timeout 600 python tools/dev/stage1_once.py c3 > gpurun_out/s1_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:s1_" -c 16 -o gpurun_out/prof_stage1_c3 -f python tools/dev/stage1_once.py c3 > gpurun_out/ncu_s1.log 2>&1; echo "stage1 ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k "regex:s1_|wiener" --log-file gpurun_out/s1w_launches.csv python tools/dev/stage1_once.py c3 > /dev/null 2>&1; echo "launch rc=$?"
