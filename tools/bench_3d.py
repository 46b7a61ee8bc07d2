"""Time ccl_label_3d_async on a 256^3 volume (random voxels at density 0.3
and a smooth blob field), 6- and 26-connectivity; L2 flushed before every run.
Algorithmic bytes: 5 B/voxel (1 read + 4 written)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1708_08180_b200 as ccl  # noqa: E402

n = 256
rng = np.random.default_rng(1)
vols = {"random d=0.3": (rng.random((n, n, n)) < 0.3).astype(np.uint8)}
z, y, x = np.indices((n, n, n), dtype=np.float32) / n
field = np.sin(9 * x + 2 * np.sin(7 * z)) + np.sin(8 * y + 3 * np.cos(5 * x)) + np.sin(10 * z + 2 * np.sin(6 * y))
vols["smooth blobs"] = (field > 0.3).astype(np.uint8)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name, v in vols.items():
    t = torch.from_numpy(v).cuda()
    for conn in (6, 26):
        out = ccl.label_3d(t, conn)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ccl.label_3d(t, conn, out=out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        print(json.dumps({"volume": f"{n}^3 {name}", "conn": conn, "ms": round(ms, 4),
                          "gvox_s": round(n ** 3 / ms / 1e6, 1), "GB_s_at_5B": round(5 * n ** 3 / ms / 1e6, 1)}))
