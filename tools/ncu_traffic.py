"""Per-launch traffic of K1/K2/K3 from the r2_ncu_final.sh raw exports:
max(DRAM read + DRAM write, DRAM read + L2 write-in), printed and written to
profiles/ncu_traffic.json (bench.py's roofline.traffic)."""
import csv
import json

SC = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}


def get(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    out = {}
    for r in data:
        n = r[idx['Kernel Name']]
        key = ('k1_local_merge' if 'k_local_merge' in n else 'k2_boundary' if 'k_boundary' in n
               else 'k3_link' if 'k_link' in n else None)
        if not key:
            continue

        def f(m):
            v = float(r[idx[m]].replace(',', ''))
            return v * SC.get(units[idx[m]], 1)
        out[key] = dict(dram_read=f('dram__bytes_read.sum'), dram_write=f('dram__bytes_write.sum'),
                        l2_write_in=float(r[idx['lts__t_sectors_srcunit_tex_op_write.sum']].replace(',', '')) * 32)
    return out


def main():
    lines = ["", "## traffic accounting per launch (bytes): DRAM read + DRAM write, and DRAM read + L2 write-in (what the kernel",
             "## wrote into L2: every dirty byte reaches DRAM, at the latest when evicted after the kernel) -- the larger is 'traffic'"]
    px = 8192 * 8192
    alg = {'k1_local_merge': 1.125 * px, 'k2_boundary': None, 'k3_link': 4.125 * px}
    tr = {}
    for c in ['texture_8', 'texture_4', 'noise_8']:
        for k, v in get(f'gpurun_out/nf_full_{c}_raw.csv').items():
            t1, t2 = v['dram_read'] + v['dram_write'], v['dram_read'] + v['l2_write_in']
            a = alg[k]
            lines.append(f"{c:10s} {k:15s} dram r+w {t1 / 1e6:8.1f} MB | dram r + L2 write-in {t2 / 1e6:8.1f} MB | "
                         f"algorithmic {a / 1e6 if a else float('nan'):8.1f} MB")
            tr.setdefault(c, {})[k] = int(max(t1, t2))
    print("\n".join(lines))
    j = {"_doc": "Bytes per launch from one `ncu --set full` capture of tools/prof_run.py --evict (C3 8192x8192, "
                 "tile 1024x32, final r02 build): max(dram__bytes_read.sum + dram__bytes_write.sum, "
                 "dram__bytes_read.sum + 32 x lts__t_sectors_srcunit_tex_op_write.sum). ncu flushes caches between "
                 "kernel passes, so labels still dirty in L2 when K3 ends are missing from its dram__bytes_write; the "
                 "L2 write-in counts them. bench.py reports the entry for its workload as roofline.traffic. Source: "
                 "profiles/r02_ncu_full_summary.txt",
         "C3 8192x8192 texture": tr['texture_8'], "C3 8192x8192 texture 4-conn": tr['texture_4'],
         "C3 8192x8192 noise 0.5": tr['noise_8']}
    json.dump(j, open('profiles/ncu_traffic.json', 'w'), indent=2)


if __name__ == "__main__":
    main()
