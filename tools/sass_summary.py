"""Per-kernel SASS census of libccl.so (cuobjdump -sass): the instructions
that show which hardware paths a kernel uses -- TMA bulk-tensor stores
(UTMASTG), bulk L2 prefetches (UBLKPF), 256-bit global loads, shared / global
atomics, griddepcontrol (PDL), barriers.  Usage: python tools/sass_summary.py
[lib] [kernel-substring ...]"""
import collections
import re
import subprocess
import sys

PATS = {
    "UTMASTG (TMA bulk-tensor store)": r"\bUTMASTG\b",
    "UTMACMDFLUSH": r"\bUTMACMDFLUSH\b",
    "UBLKPF (bulk L2 prefetch)": r"\bUBLKPF\b",
    "LDG.E.ENL2.256 / LDG.*.256": r"\bLDG\.[A-Z0-9._]*256\b",
    "LDG.*.128": r"\bLDG\.[A-Z0-9._]*128\b",
    "ATOMS (shared atomics)": r"\bATOMS\b",
    "ATOMG / RED (global atomics)": r"\b(ATOMG|RED)\b",
    "BAR.SYNC": r"\bBAR\.SYNC\b",
    "ACQBULK (griddepcontrol.wait)": r"\bACQBULK\b",
    "LDL/STL (local memory)": r"\b(LDL|STL)\b",
    "MEMBAR": r"\bMEMBAR\b",
    "STG (global stores)": r"\bSTG\b",
}


def main(lib, subs):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    counts, cur, ninst = {}, None, collections.Counter()
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None or not re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            continue
        ninst[cur] += 1
        for k, p in PATS.items():
            if re.search(p, line):
                counts[cur][k] += 1
    demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
    for (mangled, c), name in zip(counts.items(), demangle):
        if subs and not any(s in name for s in subs):
            continue
        print(f"{name.split('(')[0]}  [{ninst[mangled]} SASS instructions]")
        for k in PATS:
            if c[k]:
                print(f"    {k:36s} {c[k]}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_1708_08180_b200/libccl.so", sys.argv[2:])
