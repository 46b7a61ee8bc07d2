"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per
kernel: launches, mean duration, share of the summed device time."""
import csv
import sys
from collections import defaultdict


def main(path, title):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[h]
    K, V = hdr.index('Kernel Name'), hdr.index('Metric Value')
    n, tot = defaultdict(int), defaultdict(float)
    for r in rows[h + 1:]:
        if len(r) != len(hdr):
            continue
        name = r[K].replace('void ', '').split('(')[0]
        n[name] += 1
        tot[name] += float(r[V].replace(',', '')) / 1000.0  # ns -> us
    all_t = sum(tot.values()) or 1.0
    print(f"# ncu launch list, {title}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)")
    print(f"{'kernel':60s} {'launches':>8s} {'mean_us':>9s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:60]:60s} {n[k]:8d} {tot[k] / n[k]:9.2f} {100 * tot[k] / all_t:6.1f}%")
    ccl = {k: v for k, v in tot.items() if k.startswith('ccl::')}
    s = sum(ccl.values()) or 1.0
    print("# share of the CCL step (library kernels only):")
    for k in sorted(ccl, key=lambda k: -ccl[k]):
        print(f"#   {k[:56]:56s} {100 * ccl[k] / s:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]) or "")
