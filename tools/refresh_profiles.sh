#!/bin/bash
# One GPU call: parity tests, the default bench line, its ncu launch list, and
# one `ncu --set full` capture of the four kernels (tools/prof_run.py).
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pt.log
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1 || exit 1
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-stages > gpurun_out/bench_small.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-stages > gpurun_out/ncu_bench.log 2>&1
timeout 300 python tools/prof_run.py --iters 2 > gpurun_out/pr.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(local|boundary|resolve|link)" -c 4 \
    -o gpurun_out/full_latest -f python tools/prof_run.py --iters 1 > gpurun_out/ncu_full.log 2>&1
