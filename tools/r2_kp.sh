# Run every tools/kp_<variant> harness build on C3 texture (and noise): K1 phase / K2 / K3 timings.
python tools/mkimg.py texture 8192 8192 /tmp/tex.raw
python tools/mkimg.py noise 8192 8192 /tmp/noise.raw
for v in tools/kp_*; do
  n=$(basename $v)
  timeout 120 $v /tmp/tex.raw 8192 8192 > gpurun_out/${n}_tex.txt 2>&1
  [ -n "$NOISE" ] && timeout 120 $v /tmp/noise.raw 8192 8192 > gpurun_out/${n}_noise.txt 2>&1
done
for f in gpurun_out/kp_*_tex.txt gpurun_out/kp_*_noise.txt; do
  [ -f $f ] || continue
  echo "== $f"; grep -E "x5 |K2 full|L2-resident|K3 x3 |union |run lists|convert|edges|records" $f
done
