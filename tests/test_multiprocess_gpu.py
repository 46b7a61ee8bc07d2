"""Two real processes on one GPU (world_size 2, gloo) running the N > 1 paths
through their actual pieces:

* C5-style row strips: each rank runs the CUDA strip stages of its strip
  (ccl_strip_local -> exchange -> ccl_strip_finalize, i.e. StripLabeler.local /
  .finalize) and the 4W-int send buffers are all-gathered with a gloo
  collective staged through host memory -- the same exchange StripLabeler.label
  does with NCCL over NVLink on a multi-GPU box (PAPER.md:216 / :325 lifted to
  strips: per-part labeling, then a merge of the parts' boundary labels).  Every
  rank compares its strip with the oracle's rows.
* C4 data parallel: each rank builds its own share of bench.py's frame batch
  with bench.workload(rank, world) and labels it in one batched call; every
  frame is compared with the oracle.

No rank's kernels wait on another rank's (the collective runs on the host), so
two processes sharing one GPU is a faithful test of the host logic and the
CUDA stages, not of NVLink performance.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _entry(rank, world, port, fn, args):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def _run(world, fn, *args):
    import torch.multiprocessing as mp
    mp.spawn(_entry, args=(world, _free_port(), fn, args), nprocs=world, join=True)


def _strips_case(rank, world, kind, conn):
    import torch
    import torch.distributed as dist
    import oracle
    import paper_1708_08180_b200 as ccl
    import synth
    H, W = 1200, 3100
    img = {"texture": lambda: synth.texture(H, W, seed=11, density=0.5),
           "noise": lambda: synth.noise(H, W, 0.55, seed=12),
           "serpentine": lambda: synth.serpentine(H, W)}[kind]()
    r0, r1 = ccl.strip_bounds(H, world, rank)
    lab = ccl.StripLabeler(r1 - r0, W, r0, H, world, rank, conn)
    send = lab.local(torch.from_numpy(np.ascontiguousarray(img[r0:r1])).cuda())
    # the exchange: all-gather of the send buffers (gloo, through host memory)
    host_send = send.cpu()
    parts = [torch.empty_like(host_send) for _ in range(world)]
    dist.all_gather(parts, host_send)
    lab.gathered.copy_(torch.cat(parts).cuda())
    got = lab.finalize().cpu().numpy()
    want = oracle.label_bfs(img, conn)[r0:r1]
    assert np.array_equal(got, want), f"rank {rank} {kind} conn={conn}: {int((got != want).sum())} mismatches"


@pytest.mark.parametrize("kind", ["texture", "noise", "serpentine"])
@pytest.mark.parametrize("conn", [4, 8])
def test_strips_two_processes(kind, conn):
    _run(2, _strips_case, kind, conn)


def _c4_case(rank, world):
    import concurrent.futures as cf
    import torch
    import bench
    import oracle
    import paper_1708_08180_b200 as ccl
    _, imgs, _ = bench.workload("C4", None, rank, world, 8)
    distinct = min(imgs.shape[0], 32)
    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        want = list(ex.map(lambda f: oracle.label_bfs(imgs[f], 8), range(distinct)))
    out = ccl.label(torch.from_numpy(imgs).cuda(), 8).cpu().numpy()
    for f in range(imgs.shape[0]):
        assert np.array_equal(out[f], want[f % distinct]), f"rank {rank} frame {f}"


def test_c4_two_processes():
    _run(2, _c4_case)
