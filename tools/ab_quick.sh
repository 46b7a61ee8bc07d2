for k in texture upscaled texture; do
timeout 120 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --kind $k --conn 8 > gpurun_out/abq.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/abq.log').read().strip().splitlines()[-1]);print('$k', d['ms_per_step']*1e3, d['kernels_ms'], d.get('parity_vs_oracle'))" >> gpurun_out/ab.txt
done
