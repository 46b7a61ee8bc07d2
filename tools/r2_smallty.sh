# tile-height A/B on the small configs (C1 512^2, C2 2048^2 noise): the default rule picks 8 rows there
for rep in 1 2; do for c in C1 C2; do for ty in 8 16 32; do
  timeout 120 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-variants --config $c --tile-rows $ty 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c ty=$ty', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d.get('kernels_ms',{}).items()})"
done; done; done
