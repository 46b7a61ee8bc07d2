"""Small driver for ncu: label one C3-style image a few times through the
C ABI (used under `ncu`; never a bench number)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1708_08180_b200 as ccl  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="texture")
ap.add_argument("--size", type=int, default=8192)
ap.add_argument("--conn", type=int, default=8)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--tile-rows", type=int, default=0)
ap.add_argument("--evict", action="store_true",
                help="read 512 MiB after the step: that read kernel's DRAM writes are the step's dirty L2 lines")
a = ap.parse_args()
H = W = a.size
if a.kind == "texture":
    img = synth.texture(H, W, seed=3001, density=0.5)
elif a.kind == "blobs":
    img = synth.blobs(H, W, seed=3002)
elif a.kind == "noise":
    img = synth.noise(H, W, 0.5, seed=3004)
else:
    img = synth.noise(H, W, synth.percolation_density(a.conn), seed=3005)
t = torch.from_numpy(img).cuda()
ws = ccl.Workspace(1, H, W, a.conn)
out = torch.empty((H, W), dtype=torch.int32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush.fill_(1)
for _ in range(a.iters):
    flush.sum(dtype=torch.int64)  # read-only L2 flush: nothing of the earlier work stays in L2
    ccl.label(t, a.conn, out=out, workspace=ws, tile_rows=a.tile_rows)
    if a.evict:
        flush.sum(dtype=torch.int64)  # write-back of the step's dirty lines happens here
torch.cuda.synchronize()
print("ok", int(out.max().item()))
