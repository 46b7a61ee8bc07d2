"""CPU oracle for binary-image CCL -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product package ``paper_1708_08180_b200`` never imports it and shares no code
with it.

Contents
--------
* ``label_bfs``      -- O1, C flood fill (oracle/ccl_oracle.c), canonical labels.
* ``label_twopass``  -- O2, C sequential two-pass min-root union-find.
* ``brute_force``    -- O0, pure-Python transitive closure of the adjacency
                        relation, for tiny images (<= ~64 px).
* ``canonicalize``   -- SPEC.md:441-449: relabel any labeling so each class
                        carries 1 + its minimum raster index (0 stays 0).
* ``label_equal``    -- equal-value mode (NEXT-2): C flood fill with "same
                        value" adjacency, every pixel labeled with its
                        component's 0-based minimum raster index.
* ``label_3d``       -- 3D volumes (NEXT-4): C flood fill, 6- / 26-connectivity.
* ``binarize``       -- SPEC.md:50-58 threshold (>= t -> 255), for the fused
                        threshold-on-load mode.
* ``relabel_compact`` -- the 1..K renumbering of a canonical label map
                        (SPEC.md:336): k for the k-th distinct label in
                        increasing order, 0 for background.
* ``component_stats`` -- per-component area, bounding box and coordinate sums
                        of a canonical label map, components in increasing
                        label order ("size
                        and location of each dot").

Definition followed: L[p] = 0 if img[p] == 0, else
1 + min raster index of p's 4- or 8-connected foreground component
("give a unique ID to each connected region"; PAPER.md:137 the
label is a global linear index; PAPER.md:209 4-connectivity; 8-connectivity
per north_star; min-root convention SPEC.md:135, :140).

Every function here is pinned in ``tests/test_oracle.py`` against things other
than itself: SPEC/paper worked examples in ``tests/golden/``, closed forms,
``scipy.ndimage.label`` (a library routine), exhaustive brute force on tiny
shapes and invariants that fully determine the output.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ccl_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

ERRORS = {1: "null pointer", 2: "bad dimensions", 3: "image too large",
          4: "bad connectivity", 5: "out of host memory"}


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc -O2)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            sig = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
            for name in ("oracle_bfs", "oracle_twopass", "oracle_bfs_equal"):
                fn = getattr(lib, name)
                fn.argtypes = sig
                fn.restype = ctypes.c_int
            lib.oracle_bfs3d.argtypes = [ctypes.c_void_p, ctypes.c_int64] + sig[1:]
            lib.oracle_bfs3d.restype = ctypes.c_int
            lib.oracle_bfs_batched.argtypes = [ctypes.c_void_p, ctypes.c_int64] + sig[1:]
            lib.oracle_bfs_batched.restype = ctypes.c_int
            _lib = lib
    return _lib


def _as_image(img) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(img))
    if a.dtype != np.uint8:
        a = np.ascontiguousarray((a != 0).astype(np.uint8))
    return a


def _call(name: str, img, connectivity: int) -> np.ndarray:
    a = _as_image(img)
    if a.ndim != 2:
        raise ValueError("expected a 2D image")
    H, W = a.shape
    out = np.empty((H, W), dtype=np.int32)
    rc = getattr(_load(), name)(a.ctypes.data, H, W, int(connectivity), out.ctypes.data)
    if rc:
        raise ValueError(f"{name}: {ERRORS.get(rc, rc)}")
    return out


def label_bfs(img, connectivity: int = 8) -> np.ndarray:
    """O1: canonical labels by raster-seeded flood fill."""
    return _call("oracle_bfs", img, connectivity)


def label_equal(img, connectivity: int = 8) -> np.ndarray:
    """Equal-value mode (NEXT-2): every pixel labeled with the 0-based minimum
    raster index of its component of equal-valued pixels (the paper's raw
    value tests).  uint8 input,
    values compared as they are."""
    a = np.ascontiguousarray(np.asarray(img))
    if a.dtype != np.uint8 or a.ndim != 2:
        raise ValueError("expected a 2D uint8 image")
    H, W = a.shape
    out = np.empty((H, W), dtype=np.int32)
    rc = _load().oracle_bfs_equal(a.ctypes.data, H, W, int(connectivity), out.ctypes.data)
    if rc:
        raise ValueError(f"oracle_bfs_equal: {ERRORS.get(rc, rc)}")
    return out


def label_3d(vol, connectivity: int = 26) -> np.ndarray:
    """3D volumes (NEXT-4; "2D/3D grid"): canonical labels of a
    D x H x W volume, 6- or 26-connectivity, raster index (z*H + y)*W + x."""
    a = np.ascontiguousarray(np.asarray(vol))
    if a.dtype != np.uint8:
        a = np.ascontiguousarray((a != 0).astype(np.uint8))
    if a.ndim != 3:
        raise ValueError("expected a 3D volume [D,H,W]")
    D, H, W = a.shape
    out = np.empty((D, H, W), dtype=np.int32)
    rc = _load().oracle_bfs3d(a.ctypes.data, D, H, W, int(connectivity), out.ctypes.data)
    if rc:
        raise ValueError(f"oracle_bfs3d: {ERRORS.get(rc, rc)}")
    return out


def label_twopass(img, connectivity: int = 8) -> np.ndarray:
    """O2: canonical labels by sequential two-pass min-root union-find."""
    return _call("oracle_twopass", img, connectivity)


def label_bfs_batched(imgs, connectivity: int = 8) -> np.ndarray:
    a = _as_image(imgs)
    if a.ndim != 3:
        raise ValueError("expected [B,H,W]")
    B, H, W = a.shape
    out = np.empty((B, H, W), dtype=np.int32)
    rc = _load().oracle_bfs_batched(a.ctypes.data, B, H, W, int(connectivity), out.ctypes.data)
    if rc:
        raise ValueError(f"oracle_bfs_batched: {ERRORS.get(rc, rc)}")
    return out


def neighbours(y: int, x: int, H: int, W: int, connectivity: int):
    """N4 / N8 of (x, y), clipped to the image, no wrap-around."""
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            if (dy, dx) == (0, 0) or (connectivity == 4 and dy != 0 and dx != 0):
                continue
            yy, xx = y + dy, x + dx
            if 0 <= yy < H and 0 <= xx < W:
                yield yy, xx


def brute_force(img, connectivity: int = 8) -> np.ndarray:
    """O0: reachability by Warshall transitive closure of the adjacency matrix
    of foreground pixels; label = 1 + min reachable raster index.  Pure Python,
    O(n^3): tiny images only."""
    a = np.asarray(img)
    H, W = a.shape
    n = H * W
    if n > 256:
        raise ValueError("brute_force is for tiny images only")
    fg = [bool(a[p // W, p % W]) for p in range(n)]
    reach = [[i == j and fg[i] for j in range(n)] for i in range(n)]
    for p in range(n):
        if not fg[p]:
            continue
        y, x = divmod(p, W)
        for yy, xx in neighbours(y, x, H, W, connectivity):
            q = yy * W + xx
            if fg[q]:
                reach[p][q] = True
    for k in range(n):
        rk = reach[k]
        for i in range(n):
            if reach[i][k]:
                ri = reach[i]
                for j in range(n):
                    if rk[j]:
                        ri[j] = True
    out = np.zeros((H, W), dtype=np.int32)
    for p in range(n):
        if fg[p]:
            out[p // W, p % W] = 1 + min(q for q in range(n) if reach[p][q])
    return out


def canonicalize(labels) -> np.ndarray:
    """map every label class to 1 + its minimum raster index;
    label 0 (background) stays 0.  Idempotent."""
    lab = np.asarray(labels)
    flat = lab.reshape(-1).astype(np.int64)
    out = np.zeros(flat.shape, dtype=np.int32)
    fgm = flat != 0
    if fgm.any():
        vals = flat[fgm]
        pos = np.nonzero(fgm)[0]
        uniq, inv = np.unique(vals, return_inverse=True)
        first = np.full(uniq.shape, np.iinfo(np.int64).max, dtype=np.int64)
        np.minimum.at(first, inv, pos)
        out[fgm] = (first[inv] + 1).astype(np.int32)
    return out.reshape(lab.shape)


def component_stats(labels) -> dict:
    """Per-component statistics of a canonical label map [H,W] (NEXT-3).

    Definition ("the size and location of each dot"; SPEC.md:336
    renumbering 1..K in label order): for every distinct nonzero label l in
    increasing order, with P_l = {(x, y) : labels[y, x] == l}:
    area = |P_l|, x_min/x_max/y_min/y_max = min/max of the coordinates,
    sum_x / sum_y = sums of the coordinates.  Library primitives only
    (np.unique, ufunc.at)."""
    L = np.asarray(labels)
    H, W = L.shape
    ys, xs = np.nonzero(L)
    lab = L[ys, xs].astype(np.int64)
    uniq, inv, area = np.unique(lab, return_inverse=True, return_counts=True)
    K = len(uniq)
    xs = xs.astype(np.int64)
    ys = ys.astype(np.int64)
    x_min = np.full(K, np.iinfo(np.int64).max)
    y_min = np.full(K, np.iinfo(np.int64).max)
    x_max = np.full(K, -1)
    y_max = np.full(K, -1)
    np.minimum.at(x_min, inv, xs)
    np.minimum.at(y_min, inv, ys)
    np.maximum.at(x_max, inv, xs)
    np.maximum.at(y_max, inv, ys)
    sum_x = np.zeros(K, np.int64)
    sum_y = np.zeros(K, np.int64)
    np.add.at(sum_x, inv, xs)
    np.add.at(sum_y, inv, ys)
    return {"label": uniq, "area": area.astype(np.int64), "x_min": x_min, "y_min": y_min, "x_max": x_max,
            "y_max": y_max, "sum_x": sum_x, "sum_y": sum_y}


def relabel_compact(labels) -> np.ndarray:
    """The compact numbering of a label map [H,W] ("renumber
    labels to 1..K", NEXT-3): pixel p gets k if labels[p] is the k-th
    distinct nonzero label in increasing order, else 0.  Library primitive
    only (np.unique's sorted inverse)."""
    L = np.asarray(labels)
    out = np.zeros(L.shape, dtype=np.int32)
    fg = L != 0
    if fg.any():
        _, inv = np.unique(L[fg], return_inverse=True)
        out[fg] = (inv + 1).astype(np.int32)
    return out


def binarize(img, threshold: int) -> np.ndarray:
    """SPEC.md:50-58 binarize: 255 where the input >= threshold, else 0
    (dimensions preserved).  The CUDA path fuses this test into K1's load
    (ccl_label_threshold_async); its labels must equal label_bfs(binarize(img, t))."""
    a = np.asarray(img)
    if a.dtype != np.uint8:
        raise ValueError("expected uint8")
    return np.where(a >= int(threshold), np.uint8(255), np.uint8(0))
