# A/B on one box: GPU parity suite (optional), bench lines for the C3 kinds, K1 phase harness.
#   bash tools/r2_ab.sh TAG [notest]
TAG=${1:-ab}
if [ "$2" != "notest" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/${TAG}_pt.log
fi
for k in texture blobs noise perc; do
  timeout 200 python bench.py --kind $k --steps 20 --warmup 5 --no-e2e --cpu-seconds 0.5 > gpurun_out/${TAG}_bench_$k.log 2>&1
done
python - "$TAG" <<'PY' > gpurun_out/${TAG}_summary.txt
import json, sys
tag = sys.argv[1]
for k in ["texture", "blobs", "noise", "perc"]:
    try:
        d = json.loads([l for l in open(f"gpurun_out/{tag}_bench_{k}.log") if l.startswith("{")][-1])
        print(k, round(d["ms_per_step"] * 1e3, 2), "us", d["path_roofline"]["frac"], d.get("kernels_ms"), "parity", d.get("parity_vs_oracle"))
    except Exception as e:
        print(k, "FAILED", e)
PY
if [ -x tools/k1_phases ]; then
  python tools/mkimg.py texture 8192 8192 /tmp/tex.raw && timeout 300 tools/k1_phases /tmp/tex.raw 8192 8192 > gpurun_out/${TAG}_phases_tex.txt 2>&1
  python tools/mkimg.py noise 8192 8192 /tmp/noise.raw && timeout 300 tools/k1_phases /tmp/noise.raw 8192 8192 > gpurun_out/${TAG}_phases_noise.txt 2>&1
fi
cat gpurun_out/${TAG}_summary.txt
