#!/bin/bash
# quick device-time matrix over C3 kinds (no e2e / cpu baseline)
for spec in "texture 8" "blobs 8" "upscaled 8" "noise 8" "perc 4" "texture 4"; do
  set -- $spec
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --kind $1 --conn $2 > gpurun_out/bm_$1_$2.log 2>&1
done
