# device bounds asserts + loop guards (-DCCL_CHECK build in abvar/check.so) over the sanitize
# workload and the GPU parity tests (compute-sanitizer is not available on the pool)
cp paper_1708_08180_b200/libccl.so /tmp/libccl_intree.so
cp abvar/check.so paper_1708_08180_b200/libccl.so
timeout 600 python tools/sanitize_run.py > gpurun_out/check_run.txt 2>&1; echo "sanitize_run exit=$?" >> gpurun_out/check_run.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 >> gpurun_out/check_run.txt
cp /tmp/libccl_intree.so paper_1708_08180_b200/libccl.so
