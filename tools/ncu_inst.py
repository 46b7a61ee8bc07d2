"""Per-source-line instruction and stall shares from an ncu
`--page source --print-source cuda,sass --csv` export."""
import csv
import sys
from collections import defaultdict


def main(path, top=28):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == 'Line No')
    hdr = rows[h]
    I = hdr.index('Instructions Executed')
    W = hdr.index('Warp Stall Sampling (All Samples)')
    inst, st, src = defaultdict(float), defaultdict(float), {}
    cur, f = None, ''
    for r in rows[h + 1:]:
        if r and r[0] == 'File Path':
            f = r[1].split('/')[-1]
            continue
        if len(r) <= I or r[0] == 'Line No':
            continue
        if r[0]:
            cur = (f, int(r[0]))
            src[cur] = r[1]
        try:
            inst[cur] += float(r[I] or 0)
            st[cur] += float(r[W] or 0)
        except ValueError:
            pass
    ti, ts = sum(inst.values()) or 1, sum(st.values()) or 1
    print('TOTAL inst', ti, 'stall samples', ts)
    keys = sorted(set(inst) | set(st), key=lambda k: -(inst[k] / ti + st[k] / ts))
    for k in keys[:top]:
        print(f"{100*inst[k]/ti:5.1f}% inst {100*st[k]/ts:5.1f}% stall {k[0][:12]}:{k[1]}: {src.get(k,'').strip()[:75]}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 28)
