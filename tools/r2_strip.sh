# strip path checks: parity tests touching strips + the C5 bench line (k = 1), and C3 texture at TY 16 / 32
timeout 1200 python -m pytest tests -m gpu -q -k "strip or c5 or multiprocess or two_processes" 2>&1 | tail -5 > gpurun_out/r2_strip_pt.log
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-e2e --cpu-seconds 1 > gpurun_out/r2_strip_c5.log 2>&1
for ty in 16 32; do
timeout 300 python bench.py --tile-rows $ty --steps 20 --warmup 5 --no-e2e --no-variants --cpu-seconds 0.5 > gpurun_out/r2_tex_ty$ty.log 2>&1
done
