"""Attribute an ncu source export (cuda,sass) of k_local_merge to K1 phases by
line ranges of ccl_kernels.cuh (markers are source substrings)."""
import csv
import sys
from collections import defaultdict

SRC = '/root/repo/paper_1708_08180_b200/csrc/ccl_kernels.cuh'
MARKS = [('helpers', None), ('prefetch', 'void k1_prefetch'), ('row_init', 'void k1_row_init'),
         ('tile/convert', 'void k1_tile'), ('run lists', '// run lists: rs / re'),
         ('union', '// local UF.  The adjacencies'), ('flatten', 'sm.P[k] = find_r_ro(sm.P, k);'),
         ('edges', '// Alg. 1 l.34-39 for tile-edge items only (reading R7'),
         ('fpre', '// edge-root list order: exclusive prefix'), ('records', '// edge block header + column roots'),
         ('kernel loop', '__global__ void __launch_bounds__(kThreads, 3) k_local_merge'), ('after', '// ====== K2')]


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == 'Line No')
    hdr = rows[h]
    I, W = hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
    inst, st = defaultdict(float), defaultdict(float)
    cur, f = None, ''
    for r in rows:
        if r and r[0] == 'File Path':
            f = r[1]
            continue
        if len(r) <= I or r[0] in ('Line No', 'File Path', 'Function Name'):
            continue
        if r[0]:
            try:
                cur = (f, int(r[0]))
            except ValueError:
                continue
        try:
            inst[cur] += float(r[I] or 0)
            st[cur] += float(r[W] or 0)
        except (ValueError, TypeError):
            pass
    src = open(SRC).read().split('\n')
    starts = []
    for name, m in MARKS:
        ln = 1 if m is None else next((i + 1 for i, l in enumerate(src) if m in l), None)
        starts.append((name, ln))
    ti, ts = sum(inst.values()) or 1, sum(st.values()) or 1
    print(f'total warp-instructions {ti:.0f}')
    for (nm, a), (_, b) in zip(starts, starts[1:] + [('end', 10 ** 9)]):
        if a is None:
            continue
        ii = sum(v for (ff, l), v in inst.items() if ff.endswith('ccl_kernels.cuh') and a <= l < (b or 10 ** 9))
        ss = sum(v for (ff, l), v in st.items() if ff.endswith('ccl_kernels.cuh') and a <= l < (b or 10 ** 9))
        print(f'{nm:14s} inst {100 * ii / ti:5.1f}%  stall {100 * ss / ts:5.1f}%')
    oi = sum(v for (ff, l), v in inst.items() if not ff.endswith('ccl_kernels.cuh'))
    os_ = sum(v for (ff, l), v in st.items() if not ff.endswith('ccl_kernels.cuh'))
    print(f'{"intrinsics":14s} inst {100 * oi / ti:5.1f}%  stall {100 * os_ / ts:5.1f}%')


if __name__ == '__main__':
    main(sys.argv[1])
