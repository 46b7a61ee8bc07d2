"""Time ccl_component_stats_async (NEXT-3) on the C3 label map: 8192^2
texture, 8-conn, labels from the library; L2 flushed before every run.
Algorithmic bytes: 4 B/px (the label map read once)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402
import torch  # noqa: E402

import paper_1708_08180_b200 as ccl  # noqa: E402
import synth  # noqa: E402

n = 8192
img = torch.from_numpy(synth.texture(n, n, seed=3001, density=0.5)).cuda()
L = ccl.label(img, 8)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    counts, _ = ccl.component_stats(L, 1 << 20)
torch.cuda.synchronize()
ts = []
for _ in range(30):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    counts, _ = ccl.component_stats(L, 1 << 20)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = statistics.median(ts)
print(json.dumps({"what": "component_stats C3 8192x8192 texture labels", "components": int(counts[0]),
                  "ms_median": round(ms, 4), "gpx_s": round(n * n / ms / 1e6, 1),
                  "GB_s_at_4B_px": round(4 * n * n / ms / 1e6, 1)}))
ts = []
for _ in range(30):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    counts, _, rl = ccl.component_stats(L, 1 << 20, relabel=True)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = statistics.median(ts)
print(json.dumps({"what": "component_stats + 1..K relabel map, C3 8192x8192 texture labels",
                  "ms_median": round(ms, 4), "GB_s_at_8B_px": round(8 * n * n / ms / 1e6, 1)}))
