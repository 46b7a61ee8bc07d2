# tile-height A/B on the bench workloads: TYS / KINDS / CONNS env lists
for ty in ${TYS:-16 32}; do for c in ${CONNS:-8}; do for k in ${KINDS:-texture upscaled}; do
timeout 120 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --kind $k --conn $c --tile-rows $ty > gpurun_out/abv.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/abv.log').read().strip().splitlines()[-1]);print('ty$ty', 'c$c', '$k', round(d['ms_per_step']*1e3,1), {k2: round(v2*1e3,1) for k2,v2 in d['kernels_ms'].items()})" >> gpurun_out/ab.txt
done; done; done
for ty in ${TYS:-16 32}; do for cfg in ${CFGS:-C4 C2}; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --config $cfg --tile-rows $ty > gpurun_out/abv.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/abv.log').read().strip().splitlines()[-1]);print('ty$ty', '$cfg', round(d['ms_per_step']*1e3,1), d['value'], d.get('kernels_ms'))" >> gpurun_out/ab.txt
done; done
