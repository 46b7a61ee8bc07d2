"""NEXT-2: equal-value mode (the paper's raw-value comparisons, PAPER.md:104,
110, 123, 127, 294, 299): every pixel, background included, gets
the 0-based minimum raster index of its component of equal-valued pixels.
CPU: oracle.label_equal pinned by SPEC's worked examples, closed forms and a
library routine (scipy.ndimage.label per value).  GPU: ccl_label_equal_async
against the oracle."""
import numpy as np
import pytest

import oracle
import synth

from test_parity import assert_same

CONNS = (4, 8)


def scipy_equal(img, conn):
    """Per-value scipy.ndimage.label, combined and relabelled to the minimum
    raster index of each component (0-based)."""
    from scipy import ndimage
    st = ndimage.generate_binary_structure(2, 1 if conn == 4 else 2)
    out = np.full(img.shape, -1, np.int64)
    flat = np.arange(img.size).reshape(img.shape)
    for v in np.unique(img):
        lab, n = ndimage.label(img == v, structure=st)
        mins = ndimage.minimum(flat, lab, index=np.arange(1, n + 1))
        m = lab > 0
        out[m] = np.asarray(mins, np.int64)[lab[m] - 1]
    return out.astype(np.int32)


def test_spec_examples():
    # one block row [A,A,B,B,A] -> [0,0,2,2,4]
    assert oracle.label_equal(np.array([[7, 7, 3, 3, 7]], np.uint8), 4).tolist() == [[0, 0, 2, 2, 4]]
    # SPEC.md:371 4x4 image, equal-value components (SURVEY.md 8(c) pins)
    img = np.array([[1, 1, 0, 0], [0, 1, 0, 1], [0, 1, 1, 1], [1, 0, 0, 1]], np.uint8)
    assert oracle.label_equal(img, 4).ravel().tolist() == [0, 0, 2, 2, 4, 0, 2, 0, 4, 0, 0, 0, 12, 13, 13, 0]
    # 1x1 -> [0]; uniform -> all 0
    assert oracle.label_equal(np.array([[9]], np.uint8), 8).tolist() == [[0]]
    assert not oracle.label_equal(np.full((5, 6), 3, np.uint8), 4).any()


def test_closed_forms():
    cb = synth.checkerboard(6, 7)
    L4 = oracle.label_equal(cb, 4)
    assert (L4.ravel() == np.arange(42)).all()           # 4-conn: every cell alone
    L8 = oracle.label_equal(cb, 8)
    assert set(np.unique(L8).tolist()) == {0, 1}         # 8-conn: the two colours
    # binary image: foreground components coincide with the binary labels
    img = synth.noise(40, 50, 0.5, seed=3)
    for conn in CONNS:
        Lb, Le = oracle.label_bfs(img, conn), oracle.label_equal(img, conn)
        assert (Le[img != 0] == Lb[img != 0] - 1).all()


@pytest.mark.parametrize("conn", CONNS)
def test_oracle_vs_scipy(conn):
    rng = np.random.default_rng(11)
    for k in range(40):
        H, W = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        img = rng.integers(0, int(rng.integers(2, 5)), size=(H, W)).astype(np.uint8)
        assert (oracle.label_equal(img, conn) == scipy_equal(img, conn)).all(), f"case {k}"


@pytest.fixture(scope="module")
def ccl():
    import __graft_entry__
    __graft_entry__._load_build_module().build()
    import paper_1708_08180_b200 as m
    return m


@pytest.mark.gpu
@pytest.mark.parametrize("conn", CONNS)
def test_gpu_equal_vs_oracle(ccl, conn):
    import torch
    rng = np.random.default_rng(4)
    cases = [rng.integers(0, 3, size=(33, 17)).astype(np.uint8), rng.integers(0, 4, size=(257, 131)).astype(np.uint8),
             synth.noise(300, 1100, 0.5, seed=5), synth.texture(520, 530, seed=6), synth.checkerboard(48, 80),
             np.full((70, 90), 200, np.uint8), (synth.texture(1024, 2048, seed=8) // 64).astype(np.uint8)]
    for i, img in enumerate(cases):
        got = ccl.label_equal(torch.from_numpy(img).cuda(), conn).cpu().numpy()
        assert_same(got, oracle.label_equal(img, conn), f"equal case {i} {img.shape}")
    batch = np.stack([rng.integers(0, 3, size=(64, 96)).astype(np.uint8) for _ in range(3)])
    got = ccl.label_equal(torch.from_numpy(batch).cuda(), conn).cpu().numpy()
    for b in range(3):
        assert_same(got[b], oracle.label_equal(batch[b], conn), f"batch {b}")


def test_equal_abi_errors(ccl):
    lib = ccl.raw()
    assert lib.ccl_label_equal_async(None, 1, 64, 64, 5, None, None, 0, None) == 4
    assert lib.ccl_label_equal_async(None, 1, 64, 64, 8, None, None, 0, None) == 1
    assert lib.ccl_label_equal_async(None, 0, 64, 64, 8, None, None, 0, None) == 0
