#!/bin/bash
# dev: SASS opcode histogram of the integer-peak microkernels (which pipe each kind exercises)
cd /tmp && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
  -I "$(dirname "$0")/../../include" -c "$(dirname "$0")/../../paper_2103_10765_b200/csrc/int_peak.cu" -o ip.o
for k in 0 1 2 3; do
  echo "== kind $k"
  cuobjdump -sass -fun "_ZN5gbm3d15int_peak_kernelILi${k}EEEvPjijj" ip.o | grep -E "^\s+/\*[0-9a-f]+\*/" \
    | awk '{print $2}' | sed 's/\..*//' | sort | uniq -c | sort -rn | head -3
done
