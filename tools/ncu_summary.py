"""Summarise an ncu --page raw --csv export: selected metrics per kernel."""
import csv
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_warps', 'launch__waves_per_multiprocessor',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum',
        'lts__t_requests_op_atom.sum', 'lts__t_sectors_op_read.sum', 'lts__t_sectors_op_write.sum',
        'smsp__inst_executed.sum', 'lts__t_sector_hit_rate.pct']


def main(path, extra=()):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    names = [r[idx['Kernel Name']].split('(')[0].replace('void ', '') for r in data]
    print('metric'.ljust(62), ' | '.join(n[-28:] for n in names))
    for w in list(WANT) + list(extra):
        if w not in idx:
            continue
        print(w[:60].ljust(62), ' | '.join(r[idx[w]][:14].rjust(14) for r in data), units[idx[w]])


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2:])
