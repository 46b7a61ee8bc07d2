#!/bin/bash
# fused-step timelines of the abvar/tl_*.so builds (-DCCL_TIMELINE)
cp paper_1708_08180_b200/libccl.so /tmp/libccl.orig.so
for v in ${TLDIR:-abvar}/tl_*.so; do
  cp $v paper_1708_08180_b200/libccl.so
  for k in ${KINDS:-texture}; do
    echo "== $(basename $v) $k" >> gpurun_out/timeline.txt
    timeout 300 python tools/timeline.py $k >> gpurun_out/timeline.txt 2>&1
  done
done
cp /tmp/libccl.orig.so paper_1708_08180_b200/libccl.so
cat gpurun_out/timeline.txt
