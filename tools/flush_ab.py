"""L2 flush variants around one labeling step (C3 texture): the step's
device time after (a) a 512 MiB memset (dirty lines left in L2), (b) the
memset followed by a 512 MiB read (clean L2), (c) the read only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_08180_b200 as ccl  # noqa: E402
import synth  # noqa: E402

H = W = 8192
img = torch.from_numpy(synth.texture(H, W, seed=3001, density=0.5)).cuda()
ws = ccl.Workspace(1, H, W, 8)
out = torch.empty((H, W), dtype=torch.int32, device="cuda")
a = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
b = torch.ones(512 << 20, dtype=torch.uint8, device="cuda")
modes = {"memset": lambda: a.zero_(), "memset+read": lambda: (a.zero_(), b.sum(dtype=torch.int64)),
         "read": lambda: b.sum(dtype=torch.int64)}
for rep in range(2):
    for name, fl in modes.items():
        ts = []
        for i in range(33):
            fl()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ccl.label(img, 8, out=out, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"{name:12s} {sum(ts) / len(ts):7.1f} us")
