"""NEXT-3: per-component statistics (area, bounding box, coordinate sums;
components in increasing label order).  CPU: the oracle's component_stats
pinned against an independent pixel-loop definition, closed forms and
invariants.  GPU: ccl_component_stats_async against the oracle."""
import numpy as np
import pytest

import oracle
import synth

FIELDS = ("label", "area", "x_min", "y_min", "x_max", "y_max", "sum_x", "sum_y")


def loop_stats(L):
    """The definition written out pixel by pixel (tiny images only)."""
    acc = {}
    H, W = L.shape
    for y in range(H):
        for x in range(W):
            l = int(L[y, x])
            if l == 0:
                continue
            a = acc.setdefault(l, [0, W, H, -1, -1, 0, 0])
            a[0] += 1
            a[1] = min(a[1], x)
            a[2] = min(a[2], y)
            a[3] = max(a[3], x)
            a[4] = max(a[4], y)
            a[5] += x
            a[6] += y
    keys = sorted(acc)
    return {"label": keys, "area": [acc[k][0] for k in keys], "x_min": [acc[k][1] for k in keys],
            "y_min": [acc[k][2] for k in keys], "x_max": [acc[k][3] for k in keys], "y_max": [acc[k][4] for k in keys],
            "sum_x": [acc[k][5] for k in keys], "sum_y": [acc[k][6] for k in keys]}


def same(got, want, what=""):
    for f in FIELDS:
        assert list(np.asarray(got[f]).tolist()) == list(np.asarray(want[f]).tolist()), f"{what}: field {f}"


@pytest.mark.parametrize("conn", (4, 8))
def test_oracle_stats_vs_pixel_loop(conn):
    rng = np.random.default_rng(5)
    for k in range(60):
        H, W = int(rng.integers(1, 14)), int(rng.integers(1, 14))
        img = (rng.random((H, W)) < rng.uniform(0.2, 0.8)).astype(np.uint8)
        L = oracle.label_bfs(img, conn)
        same(oracle.component_stats(L), loop_stats(L), f"random {k}")


def test_oracle_stats_closed_forms():
    # one filled rectangle x in [3, 9], y in [2, 6] of a 10 x 12 image
    img = np.zeros((10, 12), np.uint8)
    img[2:7, 3:10] = 1
    s = oracle.component_stats(oracle.label_bfs(img, 4))
    w, h = 7, 5
    assert s["label"].tolist() == [2 * 12 + 3 + 1]
    assert s["area"].tolist() == [w * h]
    assert (s["x_min"][0], s["y_min"][0], s["x_max"][0], s["y_max"][0]) == (3, 2, 9, 6)
    assert s["sum_x"][0] == h * sum(range(3, 10)) and s["sum_y"][0] == w * sum(range(2, 7))
    # 4-connected checkerboard: every foreground pixel is its own component
    cb = synth.checkerboard(6, 7)
    s = oracle.component_stats(oracle.label_bfs(cb, 4))
    ys, xs = np.nonzero(cb)
    assert s["label"].tolist() == (ys * 7 + xs + 1).tolist()
    assert set(s["area"].tolist()) == {1}
    assert s["sum_x"].tolist() == xs.tolist() and s["y_max"].tolist() == ys.tolist()
    # empty image: no components
    assert len(oracle.component_stats(np.zeros((3, 4), np.int32))["label"]) == 0


def test_oracle_stats_invariants():
    img = synth.texture(200, 300, seed=9)
    L = oracle.label_bfs(img, 8)
    s = oracle.component_stats(L)
    assert s["area"].sum() == np.count_nonzero(img)
    assert np.all(s["label"] - 1 == s["y_min"] * 300 + (s["label"] - 1) % 300)  # the root is in the top row
    assert np.all((s["x_min"] <= s["x_max"]) & (s["y_min"] <= s["y_max"]))


@pytest.fixture(scope="module")
def ccl():
    import __graft_entry__
    __graft_entry__._load_build_module().build()
    import paper_1708_08180_b200 as m
    return m


def gpu_stats(ccl, labels_np, max_components=None):
    import torch
    L = torch.from_numpy(np.ascontiguousarray(labels_np, dtype=np.int32)).cuda()
    counts, st = ccl.component_stats(L, max_components)
    return counts.cpu().numpy(), {k: v.cpu().numpy() for k, v in st.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("conn", (4, 8))
def test_gpu_stats_vs_oracle(ccl, conn):
    import torch
    cases = [synth.noise(33, 17, 0.5, seed=1), synth.texture(300, 1100, seed=5), synth.blobs(520, 530, seed=6),
             synth.checkerboard(48, 80), synth.spiral(64, 64), synth.noise(1000, 999, 0.6, seed=3),
             np.zeros((5, 7), np.uint8), np.ones((64, 4100), np.uint8)]
    for i, img in enumerate(cases):
        L = ccl.label(torch.from_numpy(img).cuda(), conn)
        want = oracle.component_stats(oracle.label_bfs(img, conn))
        counts, st = gpu_stats(ccl, L.cpu().numpy())
        K = len(want["label"])
        assert counts[0] == K, f"case {i}: {counts[0]} components, want {K}"
        same({f: st[f][0, :K] for f in FIELDS}, want, f"case {i}")


@pytest.mark.gpu
def test_gpu_stats_full_size_and_batch(ccl):
    import torch
    img = synth.texture(8192, 8192, seed=3001, density=0.5)
    L = oracle.label_bfs(img, 8)
    want = oracle.component_stats(L)
    counts, st = gpu_stats(ccl, L)
    K = len(want["label"])
    assert counts[0] == K
    same({f: st[f][0, :K] for f in FIELDS}, want, "C3 texture")
    batch = np.stack([synth.noise(100, 300, d, seed=k) for k, d in enumerate((0.2, 0.5, 0.8))])
    Lb = oracle.label_bfs_batched(batch, 8)
    counts, st = gpu_stats(ccl, Lb)
    for b in range(3):
        want = oracle.component_stats(Lb[b])
        K = len(want["label"])
        assert counts[b] == K
        same({f: st[f][b, :K] for f in FIELDS}, want, f"batch {b}")
    # truncation: only the first max_components records, the count is exact
    want = oracle.component_stats(Lb[1])
    counts, st = gpu_stats(ccl, Lb[1], max_components=5)
    assert counts[0] == len(want["label"])
    same({f: st[f][0, :5] for f in FIELDS}, {f: want[f][:5] for f in FIELDS}, "truncated")


def test_stats_abi_errors(ccl):
    lib = ccl.raw()
    assert lib.ccl_stats_workspace_bytes(1, 64, 64) >= 64 * 64 * 4
    assert lib.ccl_stats_workspace_bytes(1, 0, 64) == 0
    assert lib.ccl_component_stats_async(None, 1, 64, 64, 0, None, None, None, 0, None) == 2   # max_components < 1
    assert lib.ccl_component_stats_async(None, 1, 64, 64, 10, None, None, None, 0, None) == 1  # NULL
    assert lib.ccl_component_stats_async(None, 0, 64, 64, 10, None, None, None, 0, None) == 0  # B = 0


# ------------------------------------------------- compact 1..K relabel
def loop_relabel(L):
    """The renumbering written out: labels visited in increasing order get 1, 2, ..."""
    ids = {}
    for l in sorted({int(v) for v in np.asarray(L).ravel() if v != 0}):
        ids[l] = len(ids) + 1
    out = np.zeros(L.shape, np.int32)
    for idx, v in np.ndenumerate(L):
        if v:
            out[idx] = ids[int(v)]
    return out


@pytest.mark.parametrize("conn", (4, 8))
def test_oracle_relabel_vs_loop_and_invariants(conn):
    rng = np.random.default_rng(11)
    for k in range(60):
        H, W = int(rng.integers(1, 14)), int(rng.integers(1, 14))
        img = (rng.random((H, W)) < rng.uniform(0.2, 0.8)).astype(np.uint8)
        L = oracle.label_bfs(img, conn)
        R = oracle.relabel_compact(L)
        assert np.array_equal(R, loop_relabel(L)), f"random {k}"
        # invariants: background stays 0; equal labels <-> equal ids; order
        # preserved; the ids are exactly 1..K
        assert np.array_equal(R == 0, L == 0)
        fg = L != 0
        pairs = set(zip(L[fg].tolist(), R[fg].tolist()))
        assert len(pairs) == len({p[0] for p in pairs}) == len({p[1] for p in pairs})
        srt = sorted(pairs)
        assert [p[1] for p in srt] == list(range(1, len(srt) + 1))
    # closed form: a checkerboard under 4-connectivity (every pixel its own
    # component) renumbers to 1, 2, 3, ... along the raster order of the fg pixels
    img = synth.checkerboard(6, 7) != 0
    R = oracle.relabel_compact(oracle.label_bfs(img.astype(np.uint8), 4))
    assert R[img].tolist() == list(range(1, int(img.sum()) + 1))


@pytest.mark.gpu
def test_gpu_relabel_matches_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1708_08180_b200 as ccl
    cases = [synth.texture(1024, 2048, seed=21, density=0.5), synth.noise(600, 1100, 0.55, seed=22),
             synth.blobs(777, 1031, seed=23, rmin=4, rmax=40), synth.texture(8192, 8192, seed=3001, density=0.5)]
    for img in cases:
        for conn in (4, 8):
            lab = ccl.label(torch.from_numpy(img).cuda(), conn)
            counts, st, rl = ccl.component_stats(lab, relabel=True)
            want = oracle.relabel_compact(lab.cpu().numpy())
            assert np.array_equal(rl.cpu().numpy(), want), f"{img.shape} conn={conn}"
            assert int(counts[0]) == int(want.max())
