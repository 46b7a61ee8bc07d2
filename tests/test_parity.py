"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, bit-exact (integer work: SURVEY.md §8(c)).  Marked gpu."""
import numpy as np
import pytest

import oracle
import synth
from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

CONNS = (4, 8)


@pytest.fixture(scope="module")
def ccl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1708_08180_b200 as m
    return m


def gpu_label(ccl, img, conn, tile_rows=0):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    out = ccl.label(t, conn, tile_rows=tile_rows)
    return out.cpu().numpy()


def assert_same(got, want, what=""):
    if not np.array_equal(got, want):
        bad = np.argwhere(got != want)
        i = tuple(bad[0])
        raise AssertionError(f"{what}: {len(bad)} mismatches; first at {i}: got {got[i]} want {want[i]}")


# ------------------------------------------------------------ fixtures
@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("conn", CONNS)
def test_golden(ccl, name, conn):
    g = load_golden(name)
    assert_same(gpu_label(ccl, g["image"], conn), g[f"conn{conn}"], name)


# ---------------------------------------------------- corpus
def corpus(seed=21):
    rng = np.random.default_rng(seed)
    dens = (0.05, 0.2, 0.5, 0.8, 0.95)
    for i in range(500):
        H, W = int(rng.integers(1, 258)), int(rng.integers(1, 258))
        yield f"noise{i}", synth.noise(H, W, dens[i % 5], seed=2000 + i)
    for H, W in [(33, 17), (257, 131), (1, 1), (1, 5000), (5000, 1), (2, 2049), (17, 1025),
                 (31, 3073), (100, 3000), (513, 1025)]:
        for d in (0.3, 0.6):
            yield f"noise{H}x{W}d{d}", synth.noise(H, W, d, seed=H * 7 + W)
    yield "spiral", synth.spiral(200, 1500)
    yield "serpentine", synth.serpentine(130, 2100)
    yield "checker", synth.checkerboard(70, 2050)
    yield "vstripes", synth.stripes(40, 2048, 2, True)
    yield "hstripes", synth.stripes(40, 2048, 2, False)
    yield "diag", synth.diagonal(300, 1300)
    yield "antidiag", synth.diagonal(1300, 1300, anti=True)
    yield "blobs", synth.blobs(700, 2500, seed=3)
    yield "texture", synth.texture(600, 2100, seed=4, density=0.5)
    yield "uniform", synth.uniform(50, 2100)
    yield "empty", np.zeros((50, 2100), np.uint8)


@pytest.mark.parametrize("tile_rows", [0, 16])  # 0: default rule (8-row tiles for these small images)
@pytest.mark.parametrize("conn", CONNS)
def test_corpus(ccl, conn, tile_rows):
    n = 0
    for name, img in corpus():
        assert_same(gpu_label(ccl, img, conn, tile_rows=tile_rows), oracle.label_bfs(img, conn),
                    f"{name} conn{conn} tile_rows={tile_rows}")
        n += 1
    assert n >= 500


@pytest.mark.parametrize("conn", CONNS)
def test_mixed_nonzero_values(ccl, conn):
    # reading R1: any nonzero byte is foreground
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, size=(300, 2100)).astype(np.uint8)
    img[rng.random(img.shape) < 0.45] = 0
    assert_same(gpu_label(ccl, img, conn), oracle.label_bfs(img, conn))


# ------------------------------------------- exhaustive tiny shapes, batched
def all_images(H, W):
    n = H * W
    codes = np.arange(1 << n, dtype=np.int64)
    return (((codes[:, None] >> np.arange(n)) & 1) * 255).astype(np.uint8).reshape(-1, H, W)


@pytest.mark.parametrize("shape", [(4, 4), (2, 8), (8, 2), (1, 16), (16, 1), (3, 5), (5, 3)])
@pytest.mark.parametrize("conn", CONNS)
def test_exhaustive_batched(ccl, shape, conn):
    import torch
    imgs = all_images(*shape)
    got = ccl.label(torch.from_numpy(imgs).cuda(), conn).cpu().numpy()
    assert_same(got, oracle.label_bfs_batched(imgs, conn), f"exhaustive {shape}")


@pytest.mark.parametrize("tile_rows", [8, 16])
@pytest.mark.parametrize("conn", CONNS)
def test_exhaustive_tile_corner_windows(ccl, tile_rows, conn):
    """Every 4x4 binary window placed across a tile corner (columns 1022..1025,
    rows TY-2..TY+1) of an otherwise empty image: exercises every K2 crossing
    case, including both diagonals through the corner (SURVEY.md §8(c) pin 5)."""
    import torch
    H, W = tile_rows + 4, 1030
    wy, wx = tile_rows - 2, 1022
    small = all_images(4, 4)
    want_small = oracle.label_bfs_batched(small, conn)
    B = small.shape[0]
    big = torch.zeros((B, H, W), dtype=torch.uint8, device="cuda")
    big[:, wy:wy + 4, wx:wx + 4] = torch.from_numpy(small).cuda()
    out = ccl.label(big, conn, tile_rows=tile_rows)
    win = out[:, wy:wy + 4, wx:wx + 4].cpu().numpy().astype(np.int64)
    outside = int(out.ne(0).sum().item()) - int((out[:, wy:wy + 4, wx:wx + 4] != 0).sum().item())
    assert outside == 0
    # translate small-image canonical labels to big-image raster indices
    ws = want_small.astype(np.int64)
    r = np.where(ws > 0, ws - 1, 0)
    want = np.where(ws > 0, (wy + r // 4) * W + wx + r % 4 + 1, 0)
    assert_same(win, want, "corner windows")


# ------------------------------------------------------- paper-size configs
@pytest.mark.parametrize("conn", CONNS)
def test_c1_512_noise(ccl, conn):
    img = synth.noise(512, 512, 0.5, seed=1)
    assert_same(gpu_label(ccl, img, conn), oracle.label_bfs(img, conn), "C1")


@pytest.mark.parametrize("conn", CONNS)
def test_c2_2048_density_sweep(ccl, conn):
    for k, d in enumerate([0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]):
        img = synth.noise(2048, 2048, d, seed=101 + k)
        assert_same(gpu_label(ccl, img, conn), oracle.label_bfs(img, conn), f"C2 d={d}")


@pytest.mark.parametrize("kind", ["texture", "blobs", "upscaled", "noise_perc"])
@pytest.mark.parametrize("conn", CONNS)
def test_c3_8192(ccl, kind, conn):
    if kind == "texture":
        img = synth.texture(8192, 8192, seed=3001, density=0.5)
    elif kind == "blobs":
        img = synth.blobs(8192, 8192, seed=3002)
    elif kind == "upscaled":
        img = synth.upscaled(8192, 8192, seed=3003)
    else:
        img = synth.noise(8192, 8192, synth.percolation_density(conn), seed=3005)
    assert_same(gpu_label(ccl, img, conn), oracle.label_bfs(img, conn), f"C3 {kind}")


@pytest.mark.parametrize("conn", CONNS)
def test_c3_tile_rows_32(ccl, conn):
    # 32-row tiles: 2048 tiles over a persistent grid of ~740 blocks, so every
    # block takes several tiles (the L2 bulk prefetch of its next tile), and a
    # noise band that overflows the 3456-run shared-memory cap (scratch path)
    img = synth.texture(8192, 8192, seed=3001, density=0.5)
    img[4096:4160] = synth.noise(64, 8192, 0.5, seed=7)
    assert_same(gpu_label(ccl, img, conn, tile_rows=32), oracle.label_bfs(img, conn), "C3 texture, tile_rows=32")


def test_c4_frames_sampled(ccl):
    """C4 at full size (1024 x 1080x1920, one batched call, as bench times it):
    16 sampled frames compared element by element with the oracle."""
    import torch
    B, H, W = 1024, 1080, 1920
    pick = [0, 1, 2, 3, 4, 5, 100, 257, 511, 512, 640, 777, 900, 1000, 1022, 1023]
    imgs = torch.zeros((B, H, W), dtype=torch.uint8, device="cuda")
    host = {}
    for f in pick:
        host[f] = synth.frames(1, H, W, first=f)[0]
        imgs[f] = torch.from_numpy(host[f]).cuda()
    # the other frames: cheap noise so every frame has work
    rest = torch.randint(0, 2, (B, H, W), dtype=torch.uint8, device="cuda", generator=torch.Generator(
        device="cuda").manual_seed(0)) * 255
    mask = torch.ones(B, dtype=torch.bool, device="cuda")
    mask[pick] = False
    imgs[mask] = rest[mask]
    del rest
    out = ccl.label(imgs, 8)
    for f in pick:
        assert_same(out[f].cpu().numpy(), oracle.label_bfs(host[f], 8), f"C4 frame {f}")


# -------------------------------------------------- determinism / configs
def test_config_independence(ccl):
    # identical output for every tile configuration
    for conn in CONNS:
        img = synth.noise(1111, 3333, 0.55, seed=8)
        ref = oracle.label_bfs(img, conn)
        for ty in (8, 16, 32):
            assert_same(gpu_label(ccl, img, conn, tile_rows=ty), ref, f"tile_rows={ty}")


@pytest.mark.parametrize("conn", CONNS)
def test_run_dense_tiles_global_scratch(ccl, conn):
    # Tiles with more runs than K1's shared-memory capacity (5632 per tile:
    # period-2 stripes / checkerboards reach TY*512) take the global-scratch
    # path; mixed with ordinary tiles in one image and one batch.
    H, W = 100, 3000
    img = synth.texture(H, W, seed=21)
    img[:, 1024:2048] = synth.stripes(H, 1024, period=2)      # 512 runs per row
    img[40:72, 2048:3000] = synth.checkerboard(32, 952)       # 4-conn: 476 per row
    img[0:16, 0:1024] = synth.stripes(16, 1024, period=2, vertical=False)
    for ty in (8, 16, 32):
        assert_same(gpu_label(ccl, img, conn, tile_rows=ty), oracle.label_bfs(img, conn), f"ty={ty}")
    batch = np.stack([img, synth.checkerboard(H, W), synth.noise(H, W, 0.5, seed=5)])
    import torch
    got = ccl.label(torch.from_numpy(batch).cuda(), conn).cpu().numpy()
    assert_same(got, oracle.label_bfs_batched(batch, conn), "batch")


def test_determinism_repeated_runs(ccl):
    # byte-identical across repeated racy runs
    import torch
    img = torch.from_numpy(synth.noise(2048, 2048, 0.5927, seed=3)).cuda()
    ref = ccl.label(img, 4).cpu()
    for _ in range(20):
        assert torch.equal(ccl.label(img, 4).cpu(), ref)


def test_unaligned_and_generic_path(ccl):
    import torch
    for H, W in [(77, 1000), (64, 1030), (5, 7), (300, 2049)]:
        img = synth.noise(H, W, 0.5, seed=W)
        flat = torch.zeros(H * W + 3, dtype=torch.uint8, device="cuda")
        flat[3:] = torch.from_numpy(img.reshape(-1)).cuda()
        view = flat[3:].view(H, W)  # misaligned base pointer -> generic path
        for conn in CONNS:
            got = ccl.label(view, conn).cpu().numpy()
            assert_same(got, oracle.label_bfs(img, conn), f"unaligned {H}x{W}")


def test_c_abi_simple_entry_points(ccl):
    import ctypes
    import torch
    L = ccl.raw()
    img = synth.blobs(300, 2100, seed=5, rmin=4, rmax=30)
    t = torch.from_numpy(img).cuda()
    out = torch.empty(img.shape, dtype=torch.int32, device="cuda")
    assert L.ccl_label(ctypes.c_void_p(t.data_ptr()), 300, 2100, 8, ctypes.c_void_p(out.data_ptr())) == 0
    torch.cuda.synchronize()
    assert_same(out.cpu().numpy(), oracle.label_bfs(img, 8), "ccl_label")
    imgs = np.stack([synth.noise(40, 1100, 0.5, seed=s) for s in range(3)])
    tb = torch.from_numpy(imgs).cuda()
    ob = torch.empty(imgs.shape, dtype=torch.int32, device="cuda")
    assert L.ccl_label_batched(ctypes.c_void_p(tb.data_ptr()), 3, 40, 1100, 4,
                               ctypes.c_void_p(ob.data_ptr())) == 0
    torch.cuda.synchronize()
    assert_same(ob.cpu().numpy(), oracle.label_bfs_batched(imgs, 4), "ccl_label_batched")


def test_stages_equal_fused(ccl):
    import torch
    img = torch.from_numpy(synth.texture(1000, 3000, seed=9)).cuda()
    ws = ccl.Workspace(1, 1000, 3000, 8)
    out = torch.empty(img.shape, dtype=torch.int32, device="cuda")
    ccl.stages(img, 8, out, ws)
    assert torch.equal(out, ccl.label(img, 8))


def test_host_session_e2e(ccl):
    import torch
    imgs = np.stack([synth.texture(540, 960, seed=s, octaves=((32, 4), (8, 2), (2, 1))) for s in range(4)])
    sess = ccl.HostSession(4, 540, 960, 8)
    sess.h_image.copy_(torch.from_numpy(imgs))
    got = sess.run().numpy()
    assert_same(got, oracle.label_bfs_batched(imgs, 8), "host e2e")


def test_host_pipeline_e2e(ccl):
    # two sessions on two streams, steps enqueued back to back without syncs
    import torch
    imgs = [synth.noise(300, 700, 0.5, seed=11), synth.blobs(300, 700, seed=12)]
    pipe = ccl.HostPipeline(1, 300, 700, 8, depth=2)
    for sess, im in zip(pipe.sessions, imgs):
        sess.h_image.copy_(torch.from_numpy(im[None]))
    for i in range(6):
        pipe.enqueue(i)
    torch.cuda.synchronize()
    for sess, im in zip(pipe.sessions, imgs):
        assert_same(sess.h_labels.numpy()[0], oracle.label_bfs(im, 8), "host pipeline")


def test_degenerate(ccl):
    import torch
    for H, W in [(1, 1), (1, 2), (2, 1), (1, 1025), (1025, 1)]:
        for v in (0, 255):
            img = np.full((H, W), v, np.uint8)
            for conn in CONNS:
                assert_same(gpu_label(ccl, img, conn), oracle.label_bfs(img, conn), f"{H}x{W}={v}")
    empty = torch.empty((0, 5, 5), dtype=torch.uint8, device="cuda")
    assert ccl.label(empty, 8).shape == (0, 5, 5)


# ------------------------------------------ row-strip sharding
@pytest.mark.parametrize("conn", CONNS)
def test_strips_emulated(ccl, conn):
    """k-way strip sharding emulated on one GPU (the all-gather is a device
    copy) must equal the unsharded canonical labeling (T6 of SURVEY.md §4)."""
    import torch
    cases = [
        ("texture", synth.texture(600, 2100, seed=4, density=0.5), (1, 2, 3, 4, 8)),
        ("noise", synth.noise(257, 1031, 0.55, seed=5), (2, 5, 7)),
        ("spiral", synth.spiral(120, 300), (2, 3, 8)),
        ("serpentine", synth.serpentine(97, 2049), (2, 4, 8)),
        ("vstripes", synth.stripes(64, 1030, 2, True), (8,)),
        ("checker", synth.checkerboard(33, 1025), (4,)),
        ("uniform", synth.uniform(40, 700), (5,)),
        ("rows1", synth.noise(8, 3000, 0.6, seed=6), (8,)),
    ]
    for name, img, ks in cases:
        want = oracle.label_bfs(img, conn)
        t = torch.from_numpy(img).cuda()
        for k in ks:
            got = ccl.label_strips_emulated(t, k, conn).cpu().numpy()
            assert_same(got, want, f"strips {name} k={k}")


def test_strips_c5_shape_sampled(ccl):
    """C5-like geometry at reduced height (full width 32768): 8 strips."""
    import torch
    img = synth.texture(512, 32768, seed=5001, density=0.5)
    t = torch.from_numpy(img).cuda()
    got = ccl.label_strips_emulated(t, 8, 8).cpu().numpy()
    assert_same(got, oracle.label_bfs(img, 8), "C5-like strips")


@pytest.mark.parametrize("conn", CONNS)
def test_strips_default_tile32(ccl, conn):
    """Strips tall enough that the library's default tile height is 32 rows
    (the C5 geometry's choice) -- dense noise tiles included, whose row ranges
    meet the strip marks."""
    import torch
    H, W = 5000, 8192
    assert ccl.default_tile_rows(1, H // 2, W) == 32
    for name, img in [("texture", synth.texture(H, W, seed=41, density=0.5)),
                      ("noise", synth.noise(H, W, 0.5, seed=42)),
                      ("perc", synth.noise(H, W, synth.percolation_density(conn), seed=43))]:
        want = oracle.label_bfs(img, conn)
        t = torch.from_numpy(img).cuda()
        for k in (1, 2):
            got = ccl.label_strips_emulated(t, k, conn).cpu().numpy()
            assert_same(got, want, f"strips {name} k={k} (32-row tiles)")


@pytest.mark.parametrize("conn", CONNS)
def test_tma_widths(ccl, conn):
    """Widths that are multiples of 32 take K3's TMA half-row stores: rows
    narrower than a tile and partial last tile columns are clipped by the
    tensor map (W = 32 .. 2080), at every tile height."""
    import torch
    for W in (32, 64, 96, 992, 1056, 2080):
        for H, seed in ((37, 1), (300, 2)):
            img = synth.texture(H, W, seed=100 * W + seed, density=0.5)
            want = oracle.label_bfs(img, conn)
            t = torch.from_numpy(img).cuda()
            for ty in (8, 16, 32):
                assert_same(ccl.label(t, conn, tile_rows=ty).cpu().numpy(), want, f"{H}x{W} ty={ty}")
