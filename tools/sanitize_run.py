"""Small workload for compute-sanitizer: every entry
point on small images, results checked against the oracle.

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1708_08180_b200 as ccl  # noqa: E402
import synth  # noqa: E402

imgs = [synth.noise(40, 1100, 0.5, seed=1), synth.texture(70, 2100, seed=2), synth.checkerboard(33, 1030)]
bad = 0
for img in imgs:
    t = torch.from_numpy(img).cuda()
    for conn in (4, 8):
        want = oracle.label_bfs(img, conn)
        for ty in (8, 16, 32):
            bad += not np.array_equal(ccl.label(t, conn, tile_rows=ty).cpu().numpy(), want)
        for m in ("uf", "line_uf", "le"):
            bad += not np.array_equal(ccl.label_method(t, conn, m).cpu().numpy(), want)
        bad += not np.array_equal(ccl.label_equal(t, conn).cpu().numpy(), oracle.label_equal(img, conn))
        L = ccl.label(t, conn)
        counts, st = ccl.component_stats(L)
        bad += int(counts[0].item()) != len(oracle.component_stats(want)["label"])
        got = ccl.label_strips_emulated(t, 3, conn) if hasattr(ccl, "label_strips_emulated") else None
        if got is not None:
            bad += not np.array_equal(got.cpu().numpy(), want)
vol = (np.random.default_rng(3).random((9, 20, 70)) < 0.3).astype(np.uint8)
for conn in (6, 26):
    bad += not np.array_equal(ccl.label_3d(torch.from_numpy(vol).cuda(), conn).cpu().numpy(), oracle.label_3d(vol, conn))
torch.cuda.synchronize()
print("sanitize_run mismatches:", bad)
sys.exit(1 if bad else 0)
