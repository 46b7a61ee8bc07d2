"""Bit-exact parity at the BASELINE.json full sizes, on the exact inputs and
launch configurations bench.py times (north_star: "bit-exact canonical labels
against the CPU oracle on every config"; the definition is, §1
"give a unique ID to each connected region", canonical form DESIGN.md R3).

* C5 -- the single 32768 x 32768 image (2^30 labels) through the row-strip
  path: k = 1 (what bench.py --config C5 runs on one GPU) and k = 2, 4, 8
  strips emulated on one GPU (each rank's ccl_strip_local / ccl_strip_finalize
  with the all-gather as a device copy) -- every one of the 2^30 labels is
  compared with oracle.label_bfs.
* C4 -- bench.py's batch for N = 1 (1024 frames) and for every rank of N = 8
  (128 frames each), built by bench.workload itself and labeled in ONE batched
  call as the bench does; every frame is compared with the oracle of its
  source frame.
"""
import concurrent.futures as cf
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

pytestmark = pytest.mark.gpu

C5 = 32768


@pytest.fixture(scope="module")
def ccl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1708_08180_b200 as m
    return m


@pytest.fixture(scope="module")
def c5_image():
    return synth.upscaled_rows(C5, C5, 5001, 0, C5)


@pytest.fixture(scope="module")
def c5_oracle(c5_image):
    return oracle.label_bfs(c5_image, 8)


def _first_diff(got, want):
    bad = np.flatnonzero(got.ravel() != want.ravel())
    i = int(bad[0])
    return f"{bad.size} mismatches, first at raster {i}: got {got.ravel()[i]} want {want.ravel()[i]}"


def test_c5_full_strip_k1(ccl, c5_image, c5_oracle):
    """The bench's N = 1 C5 path: one StripLabeler over all 32768 rows."""
    import torch
    t = torch.from_numpy(c5_image).cuda()
    lab = ccl.StripLabeler(C5, C5, 0, C5, 1, 0, 8)
    send = lab.local(t)
    lab.gathered.copy_(send)
    got = lab.finalize().cpu().numpy()
    assert np.array_equal(got, c5_oracle), "C5 k=1: " + _first_diff(got, c5_oracle)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_c5_full_strips_emulated(ccl, c5_image, c5_oracle, k):
    """C5 split into k row strips (the N = k bench geometry), emulated on one GPU."""
    import torch
    t = torch.from_numpy(c5_image).cuda()
    got = ccl.label_strips_emulated(t, k, 8).cpu().numpy()
    del t
    torch.cuda.empty_cache()
    assert np.array_equal(got, c5_oracle), f"C5 k={k}: " + _first_diff(got, c5_oracle)


def _oracle_frames(frames, conn):
    with cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        return list(ex.map(lambda f: oracle.label_bfs(f, conn), frames))


@pytest.mark.parametrize("world", [1, 8])
def test_c4_bench_batches(ccl, world):
    """Every frame of bench.py's C4 batch for every rank of an N = world run."""
    import torch
    import bench
    conn = 8
    for rank in range(world):
        _, imgs, desc = bench.workload("C4", None, rank, world, conn)
        B = imgs.shape[0]
        distinct = min(B, 32)
        want = _oracle_frames([imgs[i] for i in range(distinct)], conn)
        out = ccl.label(torch.from_numpy(imgs).cuda(), conn).cpu().numpy()
        for f in range(B):
            assert np.array_equal(imgs[f], imgs[f % distinct])  # the batch tiles its distinct frames
            assert np.array_equal(out[f], want[f % distinct]), (
                f"C4 world={world} rank={rank} frame {f}: " + _first_diff(out[f], want[f % distinct]))
