"""Pins for the CPU oracle (oracle/): every oracle function is checked against
something other than itself -- the hand-worked fixtures in tests/golden (each
citing its SPEC/PAPER passage), closed forms, a library routine
(scipy.ndimage.label), exhaustive enumeration of tiny shapes, a brute-force
transitive closure, and invariants that fully determine the canonical output
(SURVEY.md §8(c) "What pins each part").  CPU only.
"""
import itertools

import numpy as np
import pytest
from scipy import ndimage

import oracle
import synth
from conftest import golden_names, load_golden

CONNS = (4, 8)
ORACLES = {"bfs": oracle.label_bfs, "twopass": oracle.label_twopass}


def scipy_canonical(img, conn):
    """Library cross-check: scipy's labels relabelled to
    1 + min raster index."""
    st = ndimage.generate_binary_structure(2, 1 if conn == 4 else 2)
    lab, _ = ndimage.label(np.asarray(img) != 0, structure=st)
    return oracle.canonicalize(lab)


# ---------------------------------------------------------------- fixtures
@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("which", sorted(ORACLES))
@pytest.mark.parametrize("conn", CONNS)
def test_golden(name, which, conn):
    g = load_golden(name)
    assert g["citation"], "every golden fixture must cite its passage"
    out = ORACLES[which](g["image"], conn)
    np.testing.assert_array_equal(out, g[f"conn{conn}"])


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("conn", CONNS)
def test_golden_brute_force(name, conn):
    g = load_golden(name)
    np.testing.assert_array_equal(oracle.brute_force(g["image"], conn), g[f"conn{conn}"])


def test_canonicalize_spec_examples():
    # [0,0,3,3] and [7,7,2,2] both have classes {0,1},{2,3};
    # in the +1 convention (0 reserved for background) -> [1,1,3,3].
    np.testing.assert_array_equal(oracle.canonicalize(np.array([7, 7, 2, 2])), [1, 1, 3, 3])
    np.testing.assert_array_equal(oracle.canonicalize(np.array([5, 5, 9, 9])), [1, 1, 3, 3])
    # [0,0,1,1] vs [0,0,0,1] are different partitions
    a = oracle.canonicalize(np.array([4, 4, 6, 6]))
    b = oracle.canonicalize(np.array([4, 4, 4, 6]))
    assert not np.array_equal(a, b)
    # background stays 0; idempotence
    x = np.array([0, 3, 3, 0, 8])
    c = oracle.canonicalize(x)
    np.testing.assert_array_equal(c, [0, 2, 2, 0, 5])
    np.testing.assert_array_equal(oracle.canonicalize(c), c)


# ------------------------------------------------------------- closed forms
@pytest.mark.parametrize("which", sorted(ORACLES))
@pytest.mark.parametrize("conn", CONNS)
@pytest.mark.parametrize("shape", [(1, 1), (1, 17), (17, 1), (7, 9), (33, 17)])
def test_closed_forms(which, conn, shape):
    H, W = shape
    f = ORACLES[which]
    idx = np.arange(H * W, dtype=np.int32).reshape(H, W)
    # all background -> all 0; all foreground -> all 1 (SPEC.md:301, :310 uniform)
    np.testing.assert_array_equal(f(np.zeros((H, W), np.uint8), conn), 0)
    np.testing.assert_array_equal(f(synth.uniform(H, W), conn), 1)
    # checkerboard, (0,0) foreground: 4-conn singletons L = idx+1;
    # 8-conn all foreground joined diagonally, L = 1 (when a diagonal exists).
    cb = synth.checkerboard(H, W)
    out = f(cb, conn)
    fg = cb != 0
    assert (out[~fg] == 0).all()
    if conn == 4 or min(H, W) == 1:
        np.testing.assert_array_equal(out[fg], idx[fg] + 1)
    else:
        assert (out[fg] == 1).all()
    # vertical stripes at even x: L = x + 1 (columns never touch)
    vs = synth.stripes(H, W, 2, vertical=True)
    np.testing.assert_array_equal(f(vs, conn), np.where(vs != 0, idx % W + 1, 0))
    # horizontal stripes at even y: L = y*W + 1
    hs = synth.stripes(H, W, 2, vertical=False)
    np.testing.assert_array_equal(f(hs, conn), np.where(hs != 0, (idx // W) * W + 1, 0))
    # main diagonal: 4-conn L = idx+1, 8-conn L = 1
    dg = synth.diagonal(H, W)
    want = np.where(dg != 0, idx + 1 if conn == 4 else 1, 0)
    np.testing.assert_array_equal(f(dg, conn), want)


@pytest.mark.parametrize("which", sorted(ORACLES))
@pytest.mark.parametrize("conn", CONNS)
def test_single_row_and_column_runs(which, conn):
    # 1 x W: every maximal run is a component, label = run start + 1
    # (SPEC.md:256 row-scan example generalised; connectivity is irrelevant).
    rng = np.random.default_rng(5)
    for W in (1, 2, 3, 31, 32, 33, 100):
        row = (rng.random(W) < 0.6).astype(np.uint8)
        want = np.zeros(W, np.int32)
        start = -1
        for x in range(W):
            if row[x]:
                if x == 0 or not row[x - 1]:
                    start = x
                want[x] = start + 1
        np.testing.assert_array_equal(ORACLES[which](row[None, :], conn)[0], want)
        # W x 1 column: run start index is y (raster index y*1)
        np.testing.assert_array_equal(ORACLES[which](row[:, None], conn)[:, 0], want)


@pytest.mark.parametrize("which", sorted(ORACLES))
@pytest.mark.parametrize("conn", CONNS)
def test_spiral_and_serpentine_single_component(which, conn):
    for H, W in [(5, 5), (9, 13), (31, 17), (64, 64)]:
        sp = synth.spiral(H, W)
        out = ORACLES[which](sp, conn)
        assert (out[sp != 0] == 1).all() and (out[sp == 0] == 0).all()
        sn = synth.serpentine(H, W)
        out = ORACLES[which](sn, conn)
        assert (out[sn != 0] == 1).all()


# --------------------------------------------------------- library routine
def _corpus(n=520, seed=11):
    """>= 500 images: noise at densities {0.05..0.95}, sizes in
    [1..64]^2 plus the non-multiple sizes 33x17 and 257x131, adversarial shapes."""
    rng = np.random.default_rng(seed)
    dens = (0.05, 0.2, 0.5, 0.8, 0.95)
    for i in range(n):
        H, W = int(rng.integers(1, 65)), int(rng.integers(1, 65))
        yield synth.noise(H, W, dens[i % 5], seed=1000 + i)
    yield synth.noise(33, 17, 0.5, seed=9)
    yield synth.noise(257, 131, 0.5, seed=9)
    yield synth.noise(257, 131, 0.5927, seed=10)
    yield synth.spiral(40, 33)
    yield synth.checkerboard(19, 23)
    yield synth.blobs(200, 150, seed=3, rmin=4, rmax=20)
    yield synth.texture(128, 96, seed=4, density=0.45, octaves=((32, 4), (8, 2), (2, 1)))


@pytest.mark.parametrize("conn", CONNS)
def test_against_scipy_corpus(conn):
    n = 0
    for img in _corpus():
        want = scipy_canonical(img, conn)
        np.testing.assert_array_equal(oracle.label_bfs(img, conn), want)
        np.testing.assert_array_equal(oracle.label_twopass(img, conn), want)
        n += 1
    assert n >= 500


def _gutter_mosaic(H, W):
    """All 2^(H*W) binary H x W images laid out in a mosaic separated by 1-px
    background gutters, so no two cells can touch (even diagonally)."""
    n = H * W
    codes = np.arange(1 << n, dtype=np.int64)
    bits = ((codes[:, None] >> np.arange(n)) & 1).astype(np.uint8).reshape(-1, H, W)
    per_row = 256
    rows = (len(bits) + per_row - 1) // per_row
    mosaic = np.zeros((rows * (H + 1), per_row * (W + 1)), np.uint8)
    for k in range(len(bits)):
        r, c = divmod(k, per_row)
        mosaic[r * (H + 1):r * (H + 1) + H, c * (W + 1):c * (W + 1) + W] = bits[k] * 255
    return mosaic


@pytest.mark.parametrize("shape", [(4, 4), (2, 8), (8, 2), (1, 16), (16, 1), (3, 5), (5, 3)])
def test_exhaustive_tiny_shapes_vs_scipy(shape):
    mosaic = _gutter_mosaic(*shape)
    for conn in CONNS:
        want = scipy_canonical(mosaic, conn)
        np.testing.assert_array_equal(oracle.label_bfs(mosaic, conn), want)
        np.testing.assert_array_equal(oracle.label_twopass(mosaic, conn), want)


def test_brute_force_random_tiny():
    rng = np.random.default_rng(2)
    for i in range(300):
        H, W = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        img = (rng.random((H, W)) < rng.random()).astype(np.uint8)
        for conn in CONNS:
            bf = oracle.brute_force(img, conn)
            np.testing.assert_array_equal(oracle.label_bfs(img, conn), bf)
            np.testing.assert_array_equal(oracle.label_twopass(img, conn), bf)


# --------------------------------------------------------------- invariants
def check_invariants(img, lab, conn):
    """(i) L=0 <=> background; (ii) L equal across every foreground edge;
    (iii-a) L[l-1] == l for every used label l; (iii-b) L[p] <= idx(p)+1;
    (iv) #distinct labels == #components (scipy).  (ii)+(iv) make labels a
    bijection with components; (iii) makes l-1 the minimum member."""
    img = np.asarray(img) != 0
    H, W = img.shape
    flat = lab.reshape(-1)
    assert ((flat == 0) == (~img.reshape(-1))).all()
    shifts = [(0, 1), (1, 0)] + ([(1, 1), (1, -1)] if conn == 8 else [])
    for dy, dx in shifts:
        a = lab[:H - dy, max(0, -dx):W - max(0, dx)]
        b = lab[dy:, max(0, dx):W + min(0, dx)]
        fa = img[:H - dy, max(0, -dx):W - max(0, dx)]
        fb = img[dy:, max(0, dx):W + min(0, dx)]
        both = fa & fb
        assert (a[both] == b[both]).all()
    used = np.unique(flat[flat != 0])
    assert (flat[used - 1] == used).all()
    assert (flat <= np.arange(flat.size) + 1).all()
    st = ndimage.generate_binary_structure(2, 1 if conn == 4 else 2)
    _, ncomp = ndimage.label(img, structure=st)
    assert len(used) == ncomp


@pytest.mark.parametrize("conn", CONNS)
def test_invariants_random(conn):
    for i, img in enumerate(itertools.islice(_corpus(seed=99), 120)):
        check_invariants(img, oracle.label_bfs(img, conn), conn)


def test_invariants_reject_corruptions():
    # the invariant set must reject plausible mistakes: a split, a merge and a
    # relabel-to-non-minimum of a correct labeling
    img = synth.noise(24, 24, 0.5, seed=1)
    lab = oracle.label_bfs(img, 8)
    check_invariants(img, lab, 8)
    labels = np.unique(lab[lab != 0])
    big = max(labels, key=lambda l: (lab == l).sum())
    # relabel to a non-minimum member
    bad = lab.copy()
    members = np.flatnonzero(lab.reshape(-1) == big)
    assert len(members) > 1
    bad.reshape(-1)[members] = members[-1] + 1
    with pytest.raises(AssertionError):
        check_invariants(img, bad, 8)
    # merge two components
    bad = lab.copy()
    bad[bad == labels[1]] = labels[0]
    with pytest.raises(AssertionError):
        check_invariants(img, bad, 8)
    # split one component
    bad = lab.copy()
    bad.reshape(-1)[members[-1]] = members[-1] + 1
    with pytest.raises(AssertionError):
        check_invariants(img, bad, 8)


def test_batched_is_per_image():
    imgs = np.stack([synth.noise(20, 30, 0.5, seed=s) for s in range(5)])
    out = oracle.label_bfs_batched(imgs, 8)
    for b in range(5):
        np.testing.assert_array_equal(out[b], oracle.label_bfs(imgs[b], 8))


def test_error_codes():
    with pytest.raises(ValueError, match="connectivity"):
        oracle.label_bfs(np.zeros((2, 2), np.uint8), 6)
    with pytest.raises(ValueError):
        oracle.label_twopass(np.zeros((2, 2), np.uint8), 0)
