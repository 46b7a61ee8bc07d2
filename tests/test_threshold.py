"""Fused threshold-on-load (SURVEY.md 8(f) NEXT-3 "optional fused
threshold-on-load"; SPEC.md:50-58 binarize; the paper thresholds its grey
test images): ccl_label_threshold_async labels the pixels
with value >= threshold, its K1 testing the bytes as it loads them.

CPU: the oracle's binarize pinned by SPEC.md's examples and properties; the
C-ABI's argument check.  GPU: parity with label_bfs(binarize(img, t)) on
grey-level images over the whole threshold range (both K1 SWAR variants:
t <= 128 and t > 128), several tile heights, ragged shapes.
"""
import ctypes
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


# ------------------------------------------------------------------ CPU pins
def test_binarize_spec_examples():
    # pixels [0,127,128,255], threshold 128 -> [0,0,255,255]
    got = oracle.binarize(np.array([[0, 127, 128, 255]], np.uint8), 128)
    assert got.tolist() == [[0, 0, 255, 255]]
    # all-zero image, threshold 1 -> all-zero image
    assert not oracle.binarize(np.zeros((4, 4), np.uint8), 1).any()


def test_binarize_properties():
    rng = np.random.default_rng(7)
    img = rng.integers(0, 256, size=(37, 53), dtype=np.uint8)
    for t in range(256):
        b = oracle.binarize(img, t)
        assert set(np.unique(b).tolist()) <= {0, 255}
        if t > 0:  # SPEC.md:57 idempotence for 0 < t <= 255
            assert np.array_equal(oracle.binarize(b, t), b)
        assert int((b != 0).sum()) == int((img.astype(int) >= t).sum())
    # t = 1 is the default foreground test (reading R1: nonzero); t = 0: everything
    assert np.array_equal(oracle.binarize(img, 1) != 0, img != 0)
    assert oracle.binarize(img, 0).all()


def test_threshold_abi_rejects_out_of_range():
    import paper_1708_08180_b200 as ccl
    lib = ccl._binding._lib
    for t in (-1, 256, 1000):
        rc = lib.ccl_label_threshold_async(None, 1, 4, 4, 8, t, None, None, 0, 0, None)
        assert rc == 8  # CCL_ERR_CONFIG (include/ccl.h), checked before anything else


# ----------------------------------------------------------------- GPU parity
def _grey(H, W, seed):
    """Grey-level test image: smooth ramps plus noise, every byte value present."""
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:H, 0:W]
    smooth = (128 + 60 * np.sin(x / 37.0) * np.cos(y / 23.0) + 50 * np.sin((x + 2 * y) / 101.0))
    img = np.clip(smooth + rng.normal(0, 25, size=(H, W)), 0, 255).astype(np.uint8)
    img[rng.random((H, W)) < 0.01] = 0
    img[rng.random((H, W)) < 0.01] = 255
    return img


@pytest.fixture(scope="module")
def ccl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1708_08180_b200 as m
    return m


@pytest.mark.gpu
@pytest.mark.parametrize("conn", [4, 8])
def test_threshold_parity(ccl, conn):
    import torch
    # W % 16 == 0: the vector (SWAR) load path; else the scalar one
    for (H, W, seed) in [(300, 2100, 1), (257, 3073, 2), (64, 1024, 3), (500, 4096, 4)]:
        img = _grey(H, W, seed)
        t_img = torch.from_numpy(img).cuda()
        for t in (0, 1, 2, 64, 100, 127, 128, 129, 150, 200, 254, 255):
            want = oracle.label_bfs(oracle.binarize(img, t), conn)
            got = ccl.label(t_img, conn, threshold=t).cpu().numpy()
            assert np.array_equal(got, want), f"{H}x{W} t={t} conn={conn}: {(got != want).sum()} mismatches"


@pytest.mark.gpu
@pytest.mark.parametrize("ty", [8, 16, 32])
def test_threshold_tile_heights_and_batch(ccl, ty):
    import torch
    imgs = np.stack([_grey(333, 2048, 10 + i) for i in range(3)])
    t_imgs = torch.from_numpy(imgs).cuda()
    for t in (90, 128, 170):
        got = ccl.label(t_imgs, 8, threshold=t, tile_rows=ty).cpu().numpy()
        for b in range(3):
            want = oracle.label_bfs(oracle.binarize(imgs[b], t), 8)
            assert np.array_equal(got[b], want), f"ty={ty} t={t} image {b}"


@pytest.mark.gpu
def test_threshold_one_is_default(ccl):
    """threshold 1 (nonzero) through the threshold entry equals ccl_label."""
    import torch
    img = _grey(200, 2048, 5)
    t_img = torch.from_numpy(img).cuda()
    ws = ccl.Workspace(1, 200, 2048, 8)
    out = torch.empty((200, 2048), dtype=torch.int32, device="cuda")
    lib = ccl._binding._lib
    rc = lib.ccl_label_threshold_async(ctypes.c_void_p(t_img.data_ptr()), 1, 200, 2048, 8, 1,
                                       ctypes.c_void_p(out.data_ptr()), ws.ptr(), ws.nbytes, 0,
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    assert np.array_equal(out.cpu().numpy(), ccl.label(t_img, 8).cpu().numpy())
