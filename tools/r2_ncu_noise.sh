# ncu source-level capture of K1 on C3 noise (8-conn)
timeout 300 python tools/prof_run.py --iters 1 --kind noise > gpurun_out/pr_noise.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_local" -c 1 \
    -o gpurun_out/r2_noise_k1 -f python tools/prof_run.py --iters 1 --kind noise > gpurun_out/ncu_noise.log 2>&1
ncu -i gpurun_out/r2_noise_k1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2_src_noise_k1.csv 2>/dev/null
ncu -i gpurun_out/r2_noise_k1.ncu-rep --page raw --csv > gpurun_out/r2_raw_noise_k1.csv
