"""BASELINE config C2: 2048x2048 noise at densities 0.1..0.9, 4- and
8-connectivity, one B200.  Device time per image (CUDA events, L2 flushed
before every run, 30 runs, median), Mpx/s and fraction of the 5 B/px HBM
roofline (MEASURED_PEAKS.json hbm_gbs), each output checked against the oracle.

usage: python tools/sweep_c2.py > profiles/r01_c2_sweep.md
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (parity check only)
import paper_1708_08180_b200 as ccl  # noqa: E402
import synth  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    peak = 6454.3
n = 2048
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
print(f"# C2 on one B200: {n}x{n} noise, median of 30 runs, L2 flushed per run; roofline = 5 B/px at {peak:.0f} GB/s")
print()
print("| density | conn | µs | Gpx/s | roofline frac | parity |")
print("|---|---|---|---|---|---|")
for k, d in enumerate([0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]):
    img = synth.noise(n, n, d, seed=101 + k)
    t = torch.from_numpy(img).cuda()
    for conn in (4, 8):
        ws = ccl.Workspace(1, n, n, conn)
        out = torch.empty((n, n), dtype=torch.int32, device="cuda")
        for _ in range(3):
            ccl.label(t, conn, out=out, workspace=ws)
        ok = bool(np.array_equal(out.cpu().numpy(), oracle.label_bfs(img, conn)))
        ts = []
        for _ in range(30):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ccl.label(t, conn, out=out, workspace=ws)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        print(f"| {d:.1f} | {conn} | {1e3 * ms:.1f} | {n * n / ms / 1e6:.1f} | {5 * n * n / ms / 1e6 / peak:.3f} | {ok} |")
