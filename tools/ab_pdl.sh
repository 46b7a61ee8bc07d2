for v in 1 0 1 0; do
CCL_PDL=$v timeout 120 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-stages --kind texture --conn 8 > gpurun_out/ab_pdl$v.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab_pdl$v.log').read().strip().splitlines()[-1]);print('pdl$v', d['ms_per_step']*1e3)" >> gpurun_out/ab.txt
done
