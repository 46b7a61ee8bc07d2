#!/bin/bash
# interleaved repeated A/B of abvar/*.so on one workload (REPS passes): step time only
cp paper_1708_08180_b200/libccl.so /tmp/libccl.orig.so
: > gpurun_out/abrep.txt
for rep in $(seq ${REPS:-5}); do
  for v in abvar/*.so; do
    cp $v paper_1708_08180_b200/libccl.so
    timeout 120 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-stages --no-variants --kind ${KIND:-texture} ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$(basename $v)', round(d['ms_per_step']*1e3,2))" >> gpurun_out/abrep.txt
  done
done
cp /tmp/libccl.orig.so paper_1708_08180_b200/libccl.so
python -c "
import collections, statistics
d = collections.defaultdict(list)
for l in open('gpurun_out/abrep.txt'):
    k, v = l.split(); d[k].append(float(v))
for k, v in sorted(d.items()):
    print(k, 'mean', round(statistics.mean(v), 2), 'median', round(statistics.median(v), 2), 'all', v)
"
