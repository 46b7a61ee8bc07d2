"""Aggregate an `ncu --page source --print-source cuda,sass --csv` export by
CUDA source line: instruction share and warp-stall-sample share."""
import csv
import sys
from collections import defaultdict


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == 'Line No')
    hdr = rows[h]
    I = hdr.index('Instructions Executed')
    W = hdr.index('Warp Stall Sampling (All Samples)')
    inst, stall, src = defaultdict(float), defaultdict(float), {}
    cur, fname = None, ''
    for r in rows[h + 1:]:
        if r and r[0] == 'File Path':
            fname = r[1].split('/')[-1]
            continue
        if len(r) <= I or r[0] == 'Line No':
            continue
        if r[0]:
            cur = (fname, int(r[0]))
            src[cur] = r[1]
        if cur is None:
            continue
        try:
            inst[cur] += float(r[I] or 0)
            stall[cur] += float(r[W] or 0)
        except ValueError:
            pass
    ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
    print(f'total warp-instructions {ti:.0f}, stall samples {ts:.0f}')
    for ln in sorted(stall, key=lambda k: -stall[k])[:top]:
        print(f'{100*inst[ln]/ti:5.1f}% inst {100*stall[ln]/ts:5.1f}% stall  {ln[0]}:{ln[1]}: {src.get(ln, "").strip()[:80]}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
