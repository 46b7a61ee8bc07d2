"""Debug: strip path at 32-row tiles, one case per process (argv: kind k conn)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1708_08180_b200 as ccl  # noqa: E402
import synth  # noqa: E402

kind, k, conn = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
H, W = int(os.environ.get("H", 5000)), int(os.environ.get("W", 8192))
img = {"texture": lambda: synth.texture(H, W, seed=41, density=0.5),
       "noise": lambda: synth.noise(H, W, 0.5, seed=42),
       "perc": lambda: synth.noise(H, W, synth.percolation_density(conn), seed=43)}[kind]()
t = torch.from_numpy(img).cuda()
if os.environ.get("SEND"):
    lab = ccl.StripLabeler(H, W, 0, H, 1, 0, conn)
    lab.local(t)
    torch.cuda.synchronize()
    send = lab.send.cpu().numpy()
    want = oracle.label_bfs(img, conn)
    top, bot, rep = send[:W], send[W:2 * W], send[2 * W:]
    print("top ok", np.array_equal(top, want[0]), "bottom ok", np.array_equal(bot, want[-1]))
    bad = (rep < -1) | (rep >= 2 * W)
    print("reps out of range:", int(bad.sum()), rep[bad][:8], np.flatnonzero(bad)[:8])
    fgmiss = ((send[:2 * W] != 0) & (rep < 0)).sum()
    print("fg with rep<0:", int(fgmiss))
    ex = np.flatnonzero(top != want[0])[:5]
    print("top diffs at", ex, top[ex], want[0][ex])
    sys.exit(0)
try:
    got = ccl.label_strips_emulated(t, k, conn).cpu().numpy()
    want = oracle.label_bfs(img, conn)
    print(kind, k, conn, H, W, "ok" if np.array_equal(got, want) else f"MISMATCH {(got != want).sum()}")
except Exception as e:  # noqa: BLE001
    print(kind, k, conn, H, W, "ERR", str(e).splitlines()[0])
