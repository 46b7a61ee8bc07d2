"""Aggregate an ncu source export (--page source --csv --print-source cuda,sass)
of a kernel by CUDA source-line ranges of ccl_kernels.cuh.  Only the CUDA-line
rows are summed (each aggregates its SASS).  Usage: ncu_k1_phases.py CSV
start:end:name ..."""
import csv
import sys
from collections import defaultdict


def main(path, ranges):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == 'Line No')
    hdr = rows[h]
    I = hdr.index('Instructions Executed')
    S = hdr.index('Warp Stall Sampling (All Samples)')
    inst, st = defaultdict(float), defaultdict(float)
    fname = ''
    for r in rows:
        if r and r[0] == 'File Path':
            fname = r[1].split('/')[-1]
            continue
        if not r or not r[0].isdigit():
            continue
        ln = int(r[0])
        name = 'other:' + fname
        if fname == 'ccl_kernels.cuh':
            for a, b, nm in ranges:
                if a <= ln <= b:
                    name = nm
                    break
        try:
            inst[name] += float(r[I] or 0)
            st[name] += float(r[S] or 0)
        except ValueError:
            pass
    ti, ts = sum(inst.values()), sum(st.values())
    print(f"total warp-instructions {ti:.0f}, stall samples {ts:.0f}")
    for k in sorted(inst, key=lambda k: -inst[k]):
        print(f"  {k:24s} inst {100 * inst[k] / ti:5.1f}%   stall {100 * st[k] / ts:5.1f}%")


if __name__ == '__main__':
    rr = []
    for a in sys.argv[2:]:
        x, y, n = a.split(':', 2)
        rr.append((int(x), int(y), n))
    main(sys.argv[1], rr)
