"""Timeline of fused labeling steps (library built with -DCCL_TIMELINE, e.g.
tools/build_variant.sh tl -DCCL_TIMELINE, copied over the in-tree libccl.so):
globaltimer marks of K1 / K2 / K3 relative to K1's first block, mean over
steps, L2 flushed before each step.  usage: python tools/timeline.py [kind]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_08180_b200 as ccl  # noqa: E402
import synth  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "texture"
H = W = 8192
gen = {"texture": lambda: synth.texture(H, W, seed=3001, density=0.5),
       "upscaled": lambda: synth.upscaled(H, W, seed=3003) if hasattr(synth, "upscaled") else None,
       "blobs": lambda: synth.blobs(H, W, seed=3002)}
img = torch.from_numpy(gen[kind]()).cuda()
ws = ccl.Workspace(1, H, W, 8)
out = torch.empty((H, W), dtype=torch.int32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
lib = ccl._binding._lib
fn = lib.ccl_debug_timeline
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
names = ["K1 start", "K1 end", "K2 first task", "K2 last task end", "K3 first block", "K3 past PDL wait",
         "K3 end", "K1 last publish"]
acc = [0.0] * 8
n = 0
for i in range(25):
    flush.zero_()
    torch.cuda.synchronize()
    fn(None, 1)
    ccl.label(img, 8, out=out, workspace=ws)
    torch.cuda.synchronize()
    fn(buf, 0)
    if i >= 5:
        for k in range(8):
            acc[k] += (buf[k] - buf[0]) / 1e3
        n += 1
order = sorted(range(8), key=lambda k: acc[k])
for k in order:
    print(f"{names[k]:20s} {acc[k] / n:8.2f} us")

# per-task K2 stamps (builds with -DCCL_K2_DBG=8): when did the tasks end,
# relative to K1's last publish, horizontal vs vertical
if hasattr(lib, "ccl_debug_k2_stamps") and os.environ.get("K2STAMPS"):
    # the library's task split (ccl_api.cu): 32-row tiles, horizontal boundaries
    # split over 2^sub warps while the launch stays within SMs x 40 warps
    n_h, n_v = 255 * 8, 256 * 7
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    sub = 0
    while sub < 2 and (n_h << (sub + 1)) + n_v <= sms * 40:
        sub += 1
    nh = n_h << sub
    ntask = 8192  # >= tasks of C3 at 32-row tiles
    st = torch.zeros(2 * ntask, dtype=torch.int64, device="cuda")
    lib.ccl_debug_k2_stamps.argtypes = [ctypes.c_void_p]
    lib.ccl_debug_k2_stamps(st.data_ptr())
    ts = None
    if hasattr(lib, "ccl_debug_k2_taskstat"):
        ts = torch.zeros(4 * ntask, dtype=torch.int32, device="cuda")
        lib.ccl_debug_k2_taskstat.argtypes = [ctypes.c_void_p]
        lib.ccl_debug_k2_taskstat(ts.data_ptr())
    flush.zero_()
    torch.cuda.synchronize()
    fn(None, 1)
    ccl.label(img, 8, out=out, workspace=ws)
    torch.cuda.synchronize()
    fn(buf, 0)
    lib.ccl_debug_k2_stamps(None)
    a = st.view(-1, 2).cpu().numpy().astype("float64")
    used = a[:, 1] > 0
    t0, pub = float(buf[0]), float(buf[7])
    import numpy as np
    for name, sel in (("horizontal", np.arange(len(a)) < nh), ("vertical", np.arange(len(a)) >= nh)):
        m = sel & used
        s_, e_ = (a[m, 0] - t0) / 1e3, (a[m, 1] - t0) / 1e3
        d = e_ - s_
        late = e_ > (pub - t0) / 1e3
        print(f"{name}: n={m.sum()} end p50 {np.percentile(e_, 50):.1f} p90 {np.percentile(e_, 90):.1f} max {e_.max():.1f} us;"
              f" dur p50 {np.percentile(d, 50):.2f} p90 {np.percentile(d, 90):.2f} max {d.max():.2f};"
              f" ending after K1's last publish: {late.sum()}, their dur p50 {np.percentile(d[late], 50) if late.any() else 0:.2f}"
              f" max {d[late].max() if late.any() else 0:.2f}")
    if ts is not None:
        lib.ccl_debug_k2_taskstat(None)
        c = ts.view(-1, 4).cpu().numpy()[: len(a)]
        late = used & (a[:, 1] > pub)
        early = used & ~late
        for nm, m in (("tasks ending after K1's last publish", late), ("other tasks", early)):
            if m.any():
                print(f"{nm}: n={m.sum()} union steps {c[m, 0].mean():.1f} hops {c[m, 1].mean():.1f} "
                      f"retries {c[m, 2].mean():.2f} rounds {c[m, 3].mean():.2f} | max steps {c[m, 0].max()} hops {c[m, 1].max()}")
        sp = (a[:, 1] - pub) / 1e3
        print("late tasks: flag-to-end us p50/p90/max",
              [round(float(np.percentile(sp[late], q)), 2) for q in (50, 90, 100)] if late.any() else None)
    top = np.argsort(-(a[:, 1] - a[:, 0]) * used)[:8]
    print("longest tasks (id, start, end us):", [(int(i), round((a[i, 0] - t0) / 1e3, 1), round((a[i, 1] - t0) / 1e3, 1)) for i in top])

# per-tile publish times: K1's rounds (tile t is round t // grid of the persistent grid)
if hasattr(lib, "ccl_debug_tile_pub") and os.environ.get("TILEPUB"):
    import numpy as np
    ntiles = (H // 32) * (W // 1024)
    tp = torch.zeros(ntiles, dtype=torch.int64, device="cuda")
    lib.ccl_debug_tile_pub.argtypes = [ctypes.c_void_p]
    lib.ccl_debug_tile_pub(tp.data_ptr())
    flush.zero_()
    torch.cuda.synchronize()
    fn(None, 1)
    ccl.label(img, 8, out=out, workspace=ws)
    torch.cuda.synchronize()
    fn(buf, 0)
    lib.ccl_debug_tile_pub(None)
    pub = (tp.cpu().numpy().astype("float64") - float(buf[0])) / 1e3
    grid = int(os.environ.get("K1GRID", 740))
    for r in range((ntiles + grid - 1) // grid):
        x = pub[r * grid:(r + 1) * grid]
        print(f"K1 round {r}: {len(x)} tiles published p10 {np.percentile(x, 10):.1f} p50 {np.percentile(x, 50):.1f} "
              f"p90 {np.percentile(x, 90):.1f} max {x.max():.1f} us")
