for ty in 16 8; do for cfg in C1 C2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --config $cfg --tile-rows $ty > gpurun_out/abv.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/abv.log').read().strip().splitlines()[-1]);print('ty$ty', '$cfg', round(d['ms_per_step']*1e3,1), d['value'], d.get('kernels_ms'))" >> gpurun_out/ab.txt
done; done
