for ty in 16 32 8 16 32; do
timeout 120 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --kind texture --conn 8 --tile-rows $ty > gpurun_out/abty.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/abty.log').read().strip().splitlines()[-1]);print('ty$ty', d['ms_per_step']*1e3, d['kernels_ms'])" >> gpurun_out/ab.txt
done
