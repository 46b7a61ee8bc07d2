"""Does labeling two halves of a batch on two streams overlap (K1/K2 of one
half with K3 of the other)?  Profiling aid: C4-shaped batch, device time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_08180_b200 as ccl  # noqa: E402
import synth  # noqa: E402

B, H, W = int(os.environ.get("B", "256")), 1080, 1920
base = torch.from_numpy(synth.frames(8, H, W)).cuda()
imgs = base.repeat((B + 7) // 8, 1, 1)[:B].contiguous()
out = torch.empty(imgs.shape, dtype=torch.int32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


ws_full = ccl.Workspace(B, H, W, 8)
print("one call, B=%d: %.3f ms" % (B, timed(lambda: ccl.label(imgs, 8, out=out, workspace=ws_full))))
for parts in (2, 4, 8):
    n = B // parts
    wss = [ccl.Workspace(n, H, W, 8) for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]

    def run():
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        for s in streams:
            s.wait_event(ev)
        for p in range(parts):
            s = streams[p % 2]
            with torch.cuda.stream(s):
                ccl.label(imgs[p * n:(p + 1) * n], 8, out=out[p * n:(p + 1) * n], workspace=wss[p % 2], stream=s)
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            cur.wait_event(e)

    print("%d chunks on 2 streams: %.3f ms" % (parts, timed(run)))
    nseq = [ccl.Workspace(n, H, W, 8)]

    def seq():
        for p in range(parts):
            ccl.label(imgs[p * n:(p + 1) * n], 8, out=out[p * n:(p + 1) * n], workspace=nseq[0])

    print("%d chunks, one stream:  %.3f ms" % (parts, timed(seq)))
