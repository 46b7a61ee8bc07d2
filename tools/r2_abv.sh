# A/B of prebuilt libccl variants in abvar/ on the C3 bench (copied over the in-tree library).
#   KINDS="texture noise" bash tools/r2_abv.sh
KINDS=${KINDS:-texture}
cp paper_1708_08180_b200/libccl.so /tmp/libccl.orig.so
for rep in 1 2; do
for v in abvar/*.so; do
  cp $v paper_1708_08180_b200/libccl.so
  for k in $KINDS; do
    CPU="--no-cpu-baseline"; [ -n "$PARITY" ] && [ $rep = 1 ] && CPU="--cpu-seconds 0.3"
    timeout 120 python bench.py --steps 30 --warmup 5 --no-e2e $CPU --kind $k ${BENCH_ARGS} > gpurun_out/abv.log 2>&1
    python -c "import json;d=json.loads([l for l in open('gpurun_out/abv.log') if l.startswith('{')][-1]);print('$(basename $v)', '$k', '${BENCH_ARGS}', round(d['ms_per_step']*1e3,1), {k2: round(v2*1e3,1) for k2,v2 in d['kernels_ms'].items()}, 'parity', d.get('parity_vs_oracle'))" >> gpurun_out/abv.txt 2>&1 || tail -3 gpurun_out/abv.log >> gpurun_out/abv.txt
  done
done
done
cp /tmp/libccl.orig.so paper_1708_08180_b200/libccl.so
cat gpurun_out/abv.txt
