#!/bin/bash
# One GPU call: the whole -m gpu suite, then the default bench line (with the
# variant keys) and the C5 / C4 lines.
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/suite.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config C5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --config C4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
cat gpurun_out/suite.log
for f in c3 c5 c4; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_$f.json') if l.startswith('{')][-1])
print('$f', d['ms_per_step'], d.get('path_roofline',{}).get('frac'), d['config'].get('tile'), d.get('parity_vs_oracle'), d.get('parity_vs_oracle_sampled'), d.get('clocks'))
for v in d.get('variants') or []: print('   ', v)
" || tail -5 gpurun_out/bench_$f.err; done
