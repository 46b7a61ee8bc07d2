cp paper_1708_08180_b200/libccl.so /tmp/libccl_intree.so
for v in "$@"; do cp abvar/$v.so paper_1708_08180_b200/libccl.so; echo "== $v" >> gpurun_out/b3d.log; timeout 300 python tools/bench_3d.py >> gpurun_out/b3d.log 2>&1; done
cp /tmp/libccl_intree.so paper_1708_08180_b200/libccl.so
