"""NEXT-4: 3D volumes ("2D/3D grid"), 6- and 26-connectivity.
CPU: oracle.label_3d pinned by scipy.ndimage.label (3D structures), closed
forms and brute force.  GPU: ccl_label_3d_async against the oracle."""
import itertools

import numpy as np
import pytest

import oracle

from test_parity import assert_same

CONNS = (6, 26)


def canon(lab):
    """relabel every class to 1 + its minimum raster index (0 stays 0)"""
    flat = lab.ravel()
    out = np.zeros(flat.shape, np.int32)
    first = {}
    for i, l in enumerate(flat.tolist()):
        if l and l not in first:
            first[l] = i + 1
    for i, l in enumerate(flat.tolist()):
        if l:
            out[i] = first[l]
    return out.reshape(lab.shape)


def scipy_3d(vol, conn):
    from scipy import ndimage
    st = ndimage.generate_binary_structure(3, 1 if conn == 6 else 3)
    lab, _ = ndimage.label(vol != 0, structure=st)
    return canon(lab)


@pytest.mark.parametrize("conn", CONNS)
def test_oracle_3d_vs_scipy(conn):
    rng = np.random.default_rng(13)
    for k in range(40):
        D, H, W = (int(v) for v in rng.integers(1, 12, size=3))
        vol = (rng.random((D, H, W)) < rng.uniform(0.15, 0.7)).astype(np.uint8)
        assert (oracle.label_3d(vol, conn) == scipy_3d(vol, conn)).all(), f"case {k}"


def test_oracle_3d_closed_forms():
    full = np.ones((3, 4, 5), np.uint8)
    assert (oracle.label_3d(full, 6) == 1).all()
    diag = np.zeros((4, 4, 4), np.uint8)
    for i in range(4):
        diag[i, i, i] = 1
    idx = [(i * 4 + i) * 4 + i for i in range(4)]
    assert oracle.label_3d(diag, 26)[diag != 0].tolist() == [1] * 4        # corner contacts join
    assert oracle.label_3d(diag, 6)[diag != 0].tolist() == [i + 1 for i in idx]  # faces only: singletons
    cb = (np.indices((3, 4, 5)).sum(0) % 2 == 0).astype(np.uint8)       # 3D checkerboard
    assert (oracle.label_3d(cb, 6)[cb != 0] == np.flatnonzero(cb.ravel()) + 1).all()
    assert (oracle.label_3d(cb, 26)[cb != 0] == 1).all()                 # edge contacts join


def test_oracle_3d_brute_force():
    # every 2x2x2 volume (256), transitive closure of the adjacency by hand
    for bits in range(256):
        vol = np.array([(bits >> k) & 1 for k in range(8)], np.uint8).reshape(2, 2, 2)
        for conn in CONNS:
            cells = [c for c in itertools.product(range(2), repeat=3) if vol[c]]
            lab = {c: min((z * 2 + y) * 2 + x for (z, y, x) in [c]) for c in cells}
            changed = True
            while changed:
                changed = False
                for a in cells:
                    for b in cells:
                        d = sum(abs(i - j) for i, j in zip(a, b))
                        adj = d == 1 if conn == 6 else 0 < max(abs(i - j) for i, j in zip(a, b)) <= 1
                        if adj and lab[a] != lab[b]:
                            m = min(lab[a], lab[b])
                            lab[a] = lab[b] = m
                            changed = True
            want = np.zeros((2, 2, 2), np.int32)
            for c in cells:
                want[c] = lab[c] + 1
            assert (oracle.label_3d(vol, conn) == want).all(), (bits, conn)


@pytest.fixture(scope="module")
def ccl():
    import __graft_entry__
    __graft_entry__._load_build_module().build()
    import paper_1708_08180_b200 as m
    return m


@pytest.mark.gpu
@pytest.mark.parametrize("conn", CONNS)
def test_gpu_3d_vs_oracle(ccl, conn):
    import torch
    rng = np.random.default_rng(7)
    shapes = [(1, 1, 1), (5, 7, 3), (9, 33, 65), (17, 13, 100), (40, 64, 64), (3, 200, 129)]
    for k, sh in enumerate(shapes):
        for d in (0.2, 0.35, 0.6):
            vol = (rng.random(sh) < d).astype(np.uint8)
            got = ccl.label_3d(torch.from_numpy(vol).cuda(), conn).cpu().numpy()
            assert_same(got, oracle.label_3d(vol, conn), f"3d {sh} d={d}")
    batch = (rng.random((3, 12, 20, 40)) < 0.3).astype(np.uint8)
    got = ccl.label_3d(torch.from_numpy(batch).cuda(), conn).cpu().numpy()
    for b in range(3):
        assert_same(got[b], oracle.label_3d(batch[b], conn), f"3d batch {b}")


@pytest.mark.gpu
def test_gpu_3d_large(ccl):
    import torch
    rng = np.random.default_rng(8)
    vol = (rng.random((128, 256, 256)) < 0.3).astype(np.uint8)   # near the 26-conn percolation regime
    for conn in CONNS:
        got = ccl.label_3d(torch.from_numpy(vol).cuda(), conn).cpu().numpy()
        assert_same(got, oracle.label_3d(vol, conn), f"3d 128x256x256 conn={conn}")


def test_3d_abi_errors(ccl):
    lib = ccl.raw()
    assert lib.ccl_workspace_bytes_3d(1, 4, 4, 4, 6) >= 64 * 4
    assert lib.ccl_workspace_bytes_3d(1, 4, 4, 4, 8) == 0
    assert lib.ccl_label_3d_async(None, 1, 4, 4, 4, 8, None, None, 0, None) == 4
    assert lib.ccl_label_3d_async(None, 1, 0, 4, 4, 6, None, None, 0, None) == 2
    assert lib.ccl_label_3d_async(None, 1, 4, 4, 4, 26, None, None, 0, None) == 1
    assert lib.ccl_label_3d_async(None, 0, 4, 4, 4, 26, None, None, 0, None) == 0
