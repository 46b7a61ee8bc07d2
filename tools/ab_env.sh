#!/bin/bash
# A/B over prebuilt libccl variants (abvar/<name>.so) and env settings.
# usage: tools/ab_env.sh "<name>[:ENV=VAL]" ... ; kinds from $KINDS (default texture upscaled noise)
KINDS=${KINDS:-"texture upscaled noise"}
REPS=${REPS:-2}
cp paper_1708_08180_b200/libccl.so /tmp/libccl_intree.so
for rep in $(seq $REPS); do
for spec in "$@"; do
  name=${spec%%:*}; envs=""; [[ "$spec" == *:* ]] && envs=${spec#*:}
  cp abvar/$name.so paper_1708_08180_b200/libccl.so
  for k in $KINDS; do
    env $envs timeout 120 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --kind $k --conn 8 > gpurun_out/abv.log 2>&1
    python -c "import json,sys;d=json.loads(open('gpurun_out/abv.log').read().strip().splitlines()[-1]);print('$spec', '$k', round(d['ms_per_step']*1e3,1), {k2: round(v2*1e3,1) for k2,v2 in d['kernels_ms'].items()}, d.get('parity_vs_oracle'))" >> gpurun_out/ab.txt 2>&1 || tail -3 gpurun_out/abv.log >> gpurun_out/ab.txt
  done
done
done
cp /tmp/libccl_intree.so paper_1708_08180_b200/libccl.so
