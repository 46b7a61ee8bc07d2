import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, synth, paper_1708_08180_b200 as ccl
H, W, d, conn = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
img = synth.noise(H, W, d, seed=H * 7 + W)
B, _, _ = 1, H, W
ws = ccl.Workspace(1, H, W, conn)
out = torch.empty((H, W), dtype=torch.int32, device="cuda")
t = torch.from_numpy(img).cuda()
k1, k2, k3 = ccl.stage_fns()
for nm, f in (("k1", k1), ("k2", k2), ("k3", k3)):
    print("launch", nm, flush=True)
    f(t, conn, out, ws)
    torch.cuda.synchronize()
    print("done", nm, flush=True)
print(np.array_equal(out.cpu().numpy(), oracle.label_bfs(img, conn)))
o = out.cpu().numpy(); w = oracle.label_bfs(img, conn)
bad = np.argwhere(o != w)
print("mismatches", len(bad))
for b in bad[:10]:
    y, x = b
    print((y, x), "got", o[y, x], "want", w[y, x], "img", img[y, max(0,x-3):x+4])
def al(v): return (v + 255) // 256 * 256
npx = H * W; WW = (W + 31) // 32; tx = (W + 1023) // 1024; ty = (H + 15) // 16
Gb = al(npx * 4); bb = al(H * WW * 4); rb = al(tx * ((H + 31) // 32 * 32) * 512 * 4); eb = al(tx * ((H + 7) // 8) * 1152 * 4)
buf = ws.buf.cpu().numpy()
G = buf[:npx * 4].view(np.int32)
E = buf[Gb + bb + rb: Gb + bb + rb + eb].view(np.int32).reshape(-1, 1152)
F = buf[Gb + bb + rb + eb: Gb + bb + rb + 2 * eb].view(np.int32).reshape(-1, 1152)
R = buf[Gb + bb: Gb + bb + rb].view(np.uint32).reshape(-1, 16 * 512)
for t in range(tx * ty):
    n = E[t, 0]
    print("tile", t, "n", n, "lastrow base", E[t, 1], "LC0", E[t, 2], "RC0", E[t, 34], "list", E[t, 66:66 + min(n, 8)], "F", F[t, :min(n, 8)])
    print("   R", [(int(r) & 0x7fff, int(r) >> 16) for r in R[t, :6]])
print("G[3072..3080]", G[3072:3080], "G[0:4]", G[0:4])
