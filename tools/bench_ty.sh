#!/bin/bash
for ty in 8 16 32; do for kind in texture blobs noise; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --kind $kind --tile-rows $ty > gpurun_out/bm_${kind}_ty$ty.log 2>&1
done; done
