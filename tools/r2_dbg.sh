#!/bin/bash
# strip path at 32-row tiles under the CCL_CHECK build (asserts + loop guards)
out=gpurun_out/dbg.txt; : > $out
cp paper_1708_08180_b200/libccl.so /tmp/orig.so; cp abvar/check.so paper_1708_08180_b200/libccl.so
for kind in texture noise perc; do for k in 1 2; do for c in 4 8; do
  timeout 120 python tools/dbg_strip32.py $kind $k $c 2>&1 | tail -2 >> $out
done; done; done
cp /tmp/orig.so paper_1708_08180_b200/libccl.so
cat $out
