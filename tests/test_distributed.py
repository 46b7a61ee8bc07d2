"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host logic:
bench.py's max-over-ranks timing reduction, and the row-strip exchange of
the sharded path: per-rank send buffers in the C-ABI layout
(include/ccl.h: top-row labels, bottom-row labels, same-label reps), one
all-gather, then the slot union over the gathered buffers -- the GPU kernels
are replaced here by the CPU oracle on each strip, so what is tested is the
decomposition and the exchange, not the CUDA code (that is tests/test_parity.py
::test_strips_emulated on a GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, fn, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


# ----------------------------------------------------------- bench timing
def _allreduce_case(rank, world):
    import bench
    got = bench.allreduce_max(1.0 + rank, world)
    assert got == float(world)


def test_bench_allreduce_max_gloo():
    _run(2, _allreduce_case)


# ------------------------------------------------------- strip exchange
def strip_bounds(H, k, r):
    base, extra = divmod(H, k)
    row0 = r * base + min(r, extra)
    return row0, row0 + base + (1 if r < extra else 0)


def send_buffer(labels_strip):
    """C-ABI send layout for one strip (include/ccl.h ccl_strip_local):
    [top labels | bottom labels | first slot with the same label]."""
    W = labels_strip.shape[1]
    row_pair = np.concatenate([labels_strip[0], labels_strip[-1]]).astype(np.int64)
    rep = np.full(2 * W, -1, dtype=np.int64)
    first = {}
    for s, lab in enumerate(row_pair.tolist()):
        if lab:
            first.setdefault(lab, s)
            rep[s] = first[lab]
    return np.concatenate([row_pair, rep])


def merge_slots(gathered, k, W, conn):
    """Slot union over the gathered buffers (the math of ccl_strip_finalize):
    returns {old label -> merged label (min over the slot set)}."""
    n = k * 2 * W
    parent = list(range(n))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    def union(a, b):
        a, b = find(a), find(b)
        if a != b:
            parent[max(a, b)] = min(a, b)

    blk = gathered.reshape(k, 4 * W)
    for i in range(k):
        for j in range(2 * W):
            if blk[i, j] == 0:
                continue
            union(i * 2 * W + j, i * 2 * W + int(blk[i, 2 * W + j]))
            if j >= W and i + 1 < k:
                x = j - W
                for dx in ((-1, 0, 1) if conn == 8 else (0,)):
                    if 0 <= x + dx < W and blk[i + 1, x + dx]:
                        union(i * 2 * W + j, (i + 1) * 2 * W + x + dx)
    minlab = {}
    for s in range(n):
        lab = int(blk[s // (2 * W), s % (2 * W)])
        if lab:
            r = find(s)
            minlab[r] = min(minlab.get(r, lab), lab)
    remap = {}
    for s in range(n):
        lab = int(blk[s // (2 * W), s % (2 * W)])
        if lab:
            remap[lab] = minlab[find(s)]
    return remap


def _strip_case(rank, world, H, W, conn, seed):
    import oracle
    import synth
    img = synth.noise(H, W, 0.55, seed=seed)
    r0, r1 = strip_bounds(H, world, rank)
    lab = oracle.label_bfs(img[r0:r1], conn).astype(np.int64)
    lab[lab != 0] += r0 * W          # global raster labels
    send = torch.from_numpy(send_buffer(lab))
    gathered = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(gathered, send)
    g = torch.cat(gathered).numpy()
    remap = merge_slots(g, world, W, conn)
    out = np.vectorize(lambda v: remap.get(int(v), int(v)))(lab) if lab.size else lab
    want = oracle.label_bfs(img, conn)[r0:r1]
    assert np.array_equal(out, want), f"rank {rank}: strip merge differs from the full labeling"


@pytest.mark.parametrize("conn", (4, 8))
@pytest.mark.parametrize("H,W", [(40, 37), (17, 64)])
def test_strip_exchange_gloo(conn, H, W):
    _run(2, _strip_case, H, W, conn, 7)


def test_strip_exchange_math_k_up_to_8():
    # the same decomposition, single process, k = 1..8 (all-gather = concat)
    import oracle
    import synth
    for conn in (4, 8):
        for seed, (H, W) in enumerate([(24, 31), (33, 20), (64, 9)]):
            img = synth.noise(H, W, 0.6, seed=seed)
            want = oracle.label_bfs(img, conn)
            for k in range(1, 9):
                labs, sends = [], []
                for r in range(k):
                    r0, r1 = strip_bounds(H, k, r)
                    lab = oracle.label_bfs(img[r0:r1], conn).astype(np.int64)
                    lab[lab != 0] += r0 * W
                    labs.append(lab)
                    sends.append(send_buffer(lab))
                remap = merge_slots(np.concatenate(sends), k, W, conn)
                got = np.concatenate([np.vectorize(lambda v: remap.get(int(v), int(v)))(l) for l in labs])
                assert np.array_equal(got, want), (conn, H, W, k)
