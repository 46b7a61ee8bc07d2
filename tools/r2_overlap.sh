# K1 -> K2 overlap (ready flags + early launch) on vs off, same library
for ov in 0 1; do
  for args in "--kind texture" "--kind texture --tile-rows 32" "--kind blobs" "--kind perc"; do
    CCL_K1K2_OVERLAP=$ov timeout 200 python bench.py $args --steps 30 --warmup 5 --no-e2e --no-variants --cpu-seconds 0.3 > gpurun_out/ov.log 2>&1
    python -c "import json;d=json.loads([l for l in open('gpurun_out/ov.log') if l.startswith('{')][-1]);print('overlap=$ov', '$args', round(d['ms_per_step']*1e3,1), d.get('parity_vs_oracle'))" >> gpurun_out/ov.txt 2>&1 || tail -3 gpurun_out/ov.log >> gpurun_out/ov.txt
  done
done
timeout 900 python -m pytest tests -m gpu -q -x --ignore=tests/test_fullsize.py 2>&1 | tail -3 >> gpurun_out/ov.txt
