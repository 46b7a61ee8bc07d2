# One ncu --set full capture of K1/K2/K3 (C3 texture 8-conn) with source, exported per kernel,
# plus atomic-throughput counters for 8- and 4-connectivity.
set -x
timeout 300 python tools/prof_run.py --iters 2 > gpurun_out/pr.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(local|boundary|link)" -c 3 \
    -o gpurun_out/r2_full -f python tools/prof_run.py --iters 1 > gpurun_out/ncu_full.log 2>&1
for k in k_local_merge k_boundary k_link; do
  ncu -i gpurun_out/r2_full.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > gpurun_out/r2_src_$k.csv 2>/dev/null
done
ncu -i gpurun_out/r2_full.ncu-rep --page raw --csv > gpurun_out/r2_raw.csv
M=gpu__time_duration.sum,lts__t_requests_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,l1tex__t_requests_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed.sum
for c in 8 4; do
timeout 300 ncu --metrics $M --clock-control none -k regex:"k_(local|boundary|link)" -c 6 --csv python tools/prof_run.py --iters 2 --conn $c > gpurun_out/r2_atom$c.csv 2>&1
done
