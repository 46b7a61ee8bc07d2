# K1 phase / K2 per-task timeline / K3 harness on C3 texture and noise (tools/k1_phases.cu)
set -x
python tools/mkimg.py texture 8192 8192 /tmp/tex.raw
python tools/mkimg.py noise 8192 8192 /tmp/noise.raw
timeout 300 tools/k1_phases /tmp/tex.raw 8192 8192 > gpurun_out/r2_phases_tex.txt 2>&1
timeout 300 tools/k1_phases_stats /tmp/tex.raw 8192 8192 > gpurun_out/r2_phases_tex_stats.txt 2>&1
timeout 300 tools/k1_phases /tmp/noise.raw 8192 8192 > gpurun_out/r2_phases_noise.txt 2>&1
