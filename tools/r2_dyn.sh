#!/bin/bash
# dynamic K1 tile scheduling on / off (CCL_K1_DYNAMIC), same library; parity on the first pass
: > gpurun_out/dyn.txt
for rep in 1 2; do
for d in 1 0; do
  for k in ${KINDS:-texture}; do
    CPU="--no-cpu-baseline"; [ $rep = 1 ] && CPU="--cpu-seconds 0.3"
    CCL_K1_DYNAMIC=$d timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-variants $CPU --kind $k ${BENCH_ARGS} > gpurun_out/dyn.log 2>&1
    python -c "import json;d=json.loads([l for l in open('gpurun_out/dyn.log') if l.startswith('{')][-1]);print('dyn=$d', '$k', '${BENCH_ARGS}', round(d['ms_per_step']*1e3,1), {k2: round(v2*1e3,1) for k2,v2 in d['kernels_ms'].items()}, 'parity', d.get('parity_vs_oracle'))" >> gpurun_out/dyn.txt 2>&1 || tail -3 gpurun_out/dyn.log >> gpurun_out/dyn.txt
  done
done
done
cat gpurun_out/dyn.txt
