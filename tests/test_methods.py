"""The paper's comparison methods (PAPER.md:400-410,
Table 2) through ccl_label_method_async: conventional UF, line-based UF and
label equivalence must give the same canonical labels as the oracle."""
import numpy as np
import pytest

import oracle
import synth

from test_parity import assert_same

CONNS = (4, 8)
METHODS = ("uf", "line_uf", "le", "optimized")


@pytest.fixture(scope="module")
def ccl():
    import __graft_entry__
    __graft_entry__._load_build_module().build()
    import paper_1708_08180_b200 as m
    return m


def run(ccl, img, conn, method):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    return ccl.label_method(t, conn, method).cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("conn", CONNS)
def test_methods_corpus(ccl, method, conn):
    # shapes off the {32,16} / 512 block grids, tile-corner diagonals, densities
    cases = [synth.noise(33, 17, 0.5, seed=1), synth.noise(257, 131, 0.6, seed=2), synth.noise(1, 700, 0.5, seed=3),
             synth.noise(700, 1, 0.5, seed=4), synth.texture(300, 1100, seed=5), synth.blobs(520, 530, seed=6),
             synth.spiral(64, 64), synth.checkerboard(48, 80), synth.noise(512, 512, 0.5927, seed=7)]
    for i, img in enumerate(cases):
        assert_same(run(ccl, img, conn, method), oracle.label_bfs(img, conn), f"{method} case {i} {img.shape}")


@pytest.mark.gpu
@pytest.mark.parametrize("method", ("uf", "line_uf", "le"))
def test_methods_paper_sizes(ccl, method):
    # the paper's image sizes: 512^2 .. 4096^2, natural-image stand-in
    for n in (512, 1024, 2048, 4096):
        img = synth.texture(n, n, seed=3000 + n, density=0.5)
        assert_same(run(ccl, img, 8, method), oracle.label_bfs(img, 8), f"{method} {n}^2")


@pytest.mark.gpu
def test_methods_batched(ccl):
    import torch
    batch = np.stack([synth.noise(100, 300, d, seed=k) for k, d in enumerate((0.2, 0.5, 0.8))])
    for method in ("uf", "line_uf", "le"):
        got = ccl.label_method(torch.from_numpy(batch).cuda(), 8, method).cpu().numpy()
        assert_same(got, oracle.label_bfs_batched(batch, 8), f"{method} batch")


def test_method_abi_errors(ccl):
    # argument errors are reported before any device work (no GPU needed)
    lib = ccl.raw()
    assert lib.ccl_method_workspace_bytes(1, 64, 64, 8, 1) >= 64 * 64 * 4
    assert lib.ccl_method_workspace_bytes(1, 64, 64, 8, 3) >= 2 * 64 * 64 * 4
    assert lib.ccl_method_workspace_bytes(1, 64, 64, 8, 9) == 0
    assert lib.ccl_method_workspace_bytes(1, 0, 64, 8, 1) == 0
    assert lib.ccl_label_method_async(None, 1, 64, 64, 8, 9, None, None, 0, None) == 8   # CCL_ERR_CONFIG
    assert lib.ccl_label_method_async(None, 1, 64, 64, 5, 1, None, None, 0, None) == 4   # CCL_ERR_CONNECTIVITY
    assert lib.ccl_label_method_async(None, 1, 64, 64, 8, 1, None, None, 0, None) == 1   # CCL_ERR_NULL
    assert lib.ccl_label_method_async(None, 1, 70000, 4, 8, 2, None, None, 0, None) == 2  # CCL_ERR_DIMS (grid)
    assert lib.ccl_label_method_async(None, 0, 64, 64, 8, 1, None, None, 0, None) == 0   # B = 0: no-op
