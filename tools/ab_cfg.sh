# A/B of abvar/<name>.so variants on whole bench configs: CFGS (default C1 C2 C3)
cp paper_1708_08180_b200/libccl.so /tmp/libccl_intree.so
for rep in 1 2; do for v in "$@"; do
  cp abvar/$v.so paper_1708_08180_b200/libccl.so
  for cfg in ${CFGS:-C1 C2 C3}; do
    timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --config $cfg > gpurun_out/abv.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/abv.log').read().strip().splitlines()[-1]);print('$v', '$cfg', round(d['ms_per_step']*1e3,1), {k2: round(v2*1e3,1) for k2,v2 in d['kernels_ms'].items()})" >> gpurun_out/ab.txt 2>&1 || tail -2 gpurun_out/abv.log >> gpurun_out/ab.txt
  done
done; done
cp /tmp/libccl_intree.so paper_1708_08180_b200/libccl.so
