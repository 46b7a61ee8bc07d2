set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b_smi.txt
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2b_pt.log
for k in texture blobs upscaled noise perc; do
  timeout 200 python bench.py --kind $k --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2b_bench_$k.log 2>&1
done
timeout 200 python bench.py --kind texture --tile-rows 32 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2b_bench_tex32.log 2>&1
