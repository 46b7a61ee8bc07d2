# row-range K1 (no global scratch path): GPU suite + C3 kinds at tile heights 16 and 32
timeout 1500 python -m pytest tests -m gpu -q -x --ignore=tests/test_fullsize.py 2>&1 | tail -4 > gpurun_out/rng_pt.log
for ty in 16 32; do
  for k in texture blobs upscaled noise perc; do
    timeout 200 python bench.py --kind $k --tile-rows $ty --steps 20 --warmup 5 --no-e2e --no-variants --cpu-seconds 0.3 > gpurun_out/rng.log 2>&1
    python -c "import json;d=json.loads([l for l in open('gpurun_out/rng.log') if l.startswith('{')][-1]);print('ty=$ty', '$k', round(d['ms_per_step']*1e3,1), {k2: round(v2*1e3,1) for k2,v2 in d['kernels_ms'].items()}, d.get('parity_vs_oracle'))" >> gpurun_out/rng.txt 2>&1 || tail -3 gpurun_out/rng.log >> gpurun_out/rng.txt
  done
done
