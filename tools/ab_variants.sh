# A/B of prebuilt libccl variants in abvar/ (copied over the in-tree library)
for rep in 1 2; do
for v in abvar/*.so; do
  cp $v paper_1708_08180_b200/libccl.so
  for k in texture upscaled noise; do
    timeout 120 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --kind $k --conn 8 > gpurun_out/abv.log 2>&1
    python -c "import json,sys;d=json.loads(open('gpurun_out/abv.log').read().strip().splitlines()[-1]);print('$(basename $v)', '$k', round(d['ms_per_step']*1e3,1), {k2: round(v2*1e3,1) for k2,v2 in d['kernels_ms'].items()})" >> gpurun_out/ab.txt
  done
done
done
