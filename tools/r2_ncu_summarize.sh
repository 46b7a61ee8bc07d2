#!/bin/bash
# Turn the r2_ncu_final.sh exports in gpurun_out/ into profiles/r02_ncu_full_summary.txt,
# profiles/r02_launches.txt and profiles/ncu_traffic.json (run here, not on the GPU box).
X="lts__t_requests_op_atom.sum l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum lts__t_sectors_op_atom.sum lts__t_sectors_srcunit_tex_op_write.sum l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_st.sum smsp__issue_active.avg.pct_of_peak_sustained_active"
{
  echo "# r02 ncu --set full --clock-control none (+ atomic / L2-write metrics), tools/prof_run.py --iters 1 --evict"
  echo "# C3 8192x8192, library default tile 1024x32 (final r02 build); columns: K1 k_local_merge | K2 k_boundary | K3 k_link"
  echo "# (the read-only L2 flush kernels around the step are omitted; ncu flushes caches between kernel passes, so K3's"
  echo "#  labels still dirty in L2 at its end are not in its dram__bytes_write: lts__t_sectors_srcunit_tex_op_write x 32 B"
  echo "#  = what K3 wrote into L2, all of which reaches DRAM: see the traffic accounting at the bottom)"
  for c in texture_8 texture_4 noise_8; do
    echo; echo "## $c"
    python tools/ncu_summary.py gpurun_out/nf_full_${c}_raw.csv $X | cut -c1-63,95- | awk '!seen[$1]++'
  done
} > profiles/r02_ncu_full_summary.txt
python tools/launch_list.py gpurun_out/nf_launches.csv "bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-stages --no-variants (C3 8192x8192 texture, 8-conn, tile 1024x32)" > profiles/r02_launches.txt
python tools/ncu_traffic.py >> profiles/r02_ncu_full_summary.txt
