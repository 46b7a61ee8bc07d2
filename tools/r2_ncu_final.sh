#!/bin/bash
# Evidence for the default build (C3 8192^2, library default tile height):
# ncu launch list of the bench command, and `ncu --set full` captures (8- and
# 4-connectivity, texture; 8-conn noise) with the atomic counters, each
# followed by a read-only L2 flush whose DRAM writes are the step's deferred
# write-back.  Every command first runs once without ncu.
set -x
M=lts__t_requests_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,smsp__inst_executed.sum
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-stages --no-variants"
timeout 300 $B > gpurun_out/nf_bench.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/nf_launches.csv $B > gpurun_out/nf_ncu_bench.log 2>&1
for cfg in "texture 8" "texture 4" "noise 8"; do
  set -- $cfg
  timeout 300 python tools/prof_run.py --kind $1 --conn $2 --iters 1 --evict > gpurun_out/nf_pr_$1_$2.log 2>&1 || exit 1
  timeout 900 ncu --set full --metrics $M --clock-control none --import-source on \
      -k regex:"k_local_merge|k_boundary|k_link|reduce_kernel" -c 5 \
      -o gpurun_out/nf_full_$1_$2 -f python tools/prof_run.py --kind $1 --conn $2 --iters 1 --evict > gpurun_out/nf_ncu_$1_$2.log 2>&1
done

# bring back CSV exports only (gpurun copies <= 64 MiB)
for f in gpurun_out/nf_full_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${b}_details.csv 2>/dev/null
done
ncu -i gpurun_out/nf_full_texture_8.ncu-rep --page source --csv -k regex:k_local_merge > gpurun_out/nf_src_k1_texture_8.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
