"""Seeded synthetic binary-image generators shared by the oracle tests, the GPU
parity tests and ``bench.py``.

This module holds NO labeling arithmetic: it only produces uint8 images
(0 = background, 255 = foreground).  Neither ``oracle/`` nor the CUDA package
imports the other; both consume the bytes produced here.

All generators are integer-only (splitmix64 counter hashing, integer bilinear
interpolation, integer disk tests), so the same (shape, seed) yields the same
bytes on every host.  The recipe follows SURVEY.md §8(d) "Generators", which
extends SPEC.md:41-49 (``generate``: noise / stripes / checkerboard / uniform,
splitmix-style PRNG).  The paper's own inputs (lena / peppers,
PAPER.md:366-390, Fig. 5) are not available; ``texture`` / ``blobs`` /
``upscaled`` are the "natural image" stand-ins (few large components with long
boundaries), ``noise`` near the percolation threshold is the union-find stress
case.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "GAMMA", "mix64", "noise", "texture", "blobs", "upscaled", "spiral",
    "serpentine", "checkerboard", "stripes", "diagonal", "uniform",
    "frames", "percolation_density", "upscaled_rows",
]

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

FG = np.uint8(255)


def mix64(seed: int, idx: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser applied to ``seed + (idx+1)*GAMMA`` (mod 2^64)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (idx.astype(np.uint64) + np.uint64(1)) * GAMMA
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def _density_threshold(d: float) -> np.uint64:
    if not (0.0 <= d <= 1.0):
        raise ValueError(f"density must be in [0,1], got {d}")
    return np.uint64(int(d * (1 << 24)))


def noise(H: int, W: int, density: float, seed: int, *, chunk_rows: int = 2048) -> np.ndarray:
    """i.i.d. Bernoulli(density) foreground: fg iff (mix>>40) < floor(d*2^24)."""
    _check_dims(H, W)
    out = np.empty((H, W), dtype=np.uint8)
    thr = _density_threshold(density)
    for r0 in range(0, H, chunk_rows):
        r1 = min(H, r0 + chunk_rows)
        idx = np.arange(r0 * W, r1 * W, dtype=np.uint64)
        out[r0:r1] = np.where((mix64(seed, idx) >> np.uint64(40)) < thr, FG, 0).reshape(r1 - r0, W)
    return out


def _lattice(seed: int, rows: int, cols: int) -> np.ndarray:
    idx = np.arange(rows * cols, dtype=np.uint64)
    return (mix64(seed, idx) >> np.uint64(56)).astype(np.int64).reshape(rows, cols)


_DEFAULT_OCTAVES = ((128, 4), (32, 2), (8, 1))


def _texture_values(H: int, W: int, seed: int, octaves, r0: int, r1: int) -> np.ndarray:
    """Sum over octaves of integer-bilinear lattice noise, rows [r0, r1)."""
    ys = np.arange(r0, r1, dtype=np.int64)
    xs = np.arange(W, dtype=np.int64)
    acc = np.zeros((r1 - r0, W), dtype=np.int32)
    for k, (c, w) in enumerate(octaves):
        lat = _lattice(seed * 1000003 + k, H // c + 2, W // c + 2).astype(np.int32)
        iy, fy = ys // c, (ys % c).astype(np.int32)
        ix, fx = xs // c, (xs % c).astype(np.int32)
        j0, j1 = int(iy[0]), int(iy[-1]) + 2
        # separable integer bilinear: along x on the lattice rows, then along y
        lx = lat[j0:j1, ix] * (c - fx) + lat[j0:j1, ix + 1] * fx
        rows = iy - j0
        v = (lx[rows] * (c - fy)[:, None] + lx[rows + 1] * fy[:, None]) // (c * c)
        acc += np.int32(w) * v
    return acc


def texture(H: int, W: int, seed: int, density: float = 0.5, octaves=_DEFAULT_OCTAVES,
            *, chunk_rows: int = 1024) -> np.ndarray:
    """Smooth multi-octave value noise thresholded at the exact integer quantile
    giving ``density`` foreground (few large components, long boundaries)."""
    _check_dims(H, W)
    vmax = 255 * sum(w for _, w in octaves)
    hist = np.zeros(vmax + 2, dtype=np.int64)
    for r0 in range(0, H, chunk_rows):
        r1 = min(H, r0 + chunk_rows)
        hist += np.bincount(_texture_values(H, W, seed, octaves, r0, r1).ravel(), minlength=vmax + 2)
    target = int(density * H * W)
    cum = np.cumsum(hist)
    # fg iff value < t, t the smallest value whose cumulative count reaches target
    t = int(np.searchsorted(cum, target, side="left")) if target > 0 else 0
    out = np.empty((H, W), dtype=np.uint8)
    for r0 in range(0, H, chunk_rows):
        r1 = min(H, r0 + chunk_rows)
        out[r0:r1] = np.where(_texture_values(H, W, seed, octaves, r0, r1) < t, FG, 0)
    return out


def blobs(H: int, W: int, seed: int, coverage: float = 0.35, rmin: int = 8, rmax: int = 96) -> np.ndarray:
    """Union of disks with integer centre/radius; disk count chosen so the
    expected (overlap-free) covered area is ``coverage`` of the image."""
    _check_dims(H, W)
    rmax = max(rmin, min(rmax, max(1, min(H, W) // 2)))
    rmin = min(rmin, rmax)
    mean_area = np.pi * (rmin * rmin + rmin * rmax + rmax * rmax) / 3.0
    n = max(1, int(coverage * H * W / mean_area))
    r = mix64(seed, np.arange(3 * n, dtype=np.uint64))
    cy = (r[0::3] % np.uint64(H)).astype(np.int64)
    cx = (r[1::3] % np.uint64(W)).astype(np.int64)
    rad = (rmin + (r[2::3] % np.uint64(rmax - rmin + 1))).astype(np.int64)
    out = np.zeros((H, W), dtype=np.uint8)
    for y, x, rr in zip(cy.tolist(), cx.tolist(), rad.tolist()):
        y0, y1 = max(0, y - rr), min(H, y + rr + 1)
        x0, x1 = max(0, x - rr), min(W, x + rr + 1)
        dy = np.arange(y0, y1, dtype=np.int64)[:, None] - y
        dx = np.arange(x0, x1, dtype=np.int64)[None, :] - x
        sub = out[y0:y1, x0:x1]
        sub[dy * dy + dx * dx <= rr * rr] = FG
    return out


def upscaled(H: int, W: int, seed: int, factor: int = 16, density: float = 0.5) -> np.ndarray:
    """A (H/f)x(W/f) texture nearest-neighbour upscaled by ``factor`` -- the
    paper-style resize of one base image to several sizes."""
    if H % factor or W % factor:
        raise ValueError("H and W must be multiples of factor")
    base = texture(H // factor, W // factor, seed, density, octaves=((32, 4), (8, 2), (2, 1)))
    return np.repeat(np.repeat(base, factor, axis=0), factor, axis=1)


def upscaled_rows(H: int, W: int, seed: int, r0: int, r1: int, factor: int = 16,
                  density: float = 0.5) -> np.ndarray:
    """Rows [r0, r1) of ``upscaled(H, W, seed, factor, density)`` without
    materialising the whole image (row-strip sharded gigapixel inputs, C5)."""
    if H % factor or W % factor:
        raise ValueError("H and W must be multiples of factor")
    base = texture(H // factor, W // factor, seed, density, octaves=((32, 4), (8, 2), (2, 1)))
    rows = base[np.arange(r0, r1) // factor]
    return np.repeat(rows, factor, axis=1)


def spiral(H: int, W: int) -> np.ndarray:
    """Single 1-px-wide rectangular spiral (walls separated by 1-px gaps):
    exactly one foreground component, maximal chain length."""
    _check_dims(H, W)
    out = np.zeros((H, W), dtype=np.uint8)
    dirs = ((0, 1), (1, 0), (0, -1), (-1, 0))
    y = x = d = 0
    out[0, 0] = FG

    def free(yy, xx):
        return 0 <= yy < H and 0 <= xx < W and out[yy, xx] == 0

    def far_ok(yy, xx):
        return not (0 <= yy < H and 0 <= xx < W) or out[yy, xx] == 0

    while True:
        for _ in range(2):  # go straight, else turn right once
            dy, dx = dirs[d]
            if free(y + dy, x + dx) and far_ok(y + 2 * dy, x + 2 * dx):
                break
            d = (d + 1) % 4
        else:
            return out
        dy, dx = dirs[d]
        if not (free(y + dy, x + dx) and far_ok(y + 2 * dy, x + 2 * dx)):
            return out
        y, x = y + dy, x + dx
        out[y, x] = FG


def serpentine(H: int, W: int, period: int = 2) -> np.ndarray:
    """Boustrophedon path: full rows every ``period`` rows joined alternately at
    the right and left end -- one component crossing every tile boundary."""
    _check_dims(H, W)
    out = np.zeros((H, W), dtype=np.uint8)
    out[0::period, :] = FG
    for k, y in enumerate(range(0, H - period, period)):
        x = W - 1 if k % 2 == 0 else 0
        out[y:y + period + 1, x] = FG
    return out


def checkerboard(H: int, W: int, phase: int = 0) -> np.ndarray:
    """(x+y+phase) even -> foreground; phase 0 puts (0,0) in the foreground."""
    y, x = np.indices((H, W))
    return np.where((x + y + phase) % 2 == 0, FG, 0).astype(np.uint8)


def stripes(H: int, W: int, period: int = 2, vertical: bool = True) -> np.ndarray:
    """Foreground at coordinate % period == 0 (x for vertical, y for horizontal)."""
    y, x = np.indices((H, W))
    c = x if vertical else y
    return np.where(c % period == 0, FG, 0).astype(np.uint8)


def diagonal(H: int, W: int, anti: bool = False) -> np.ndarray:
    y, x = np.indices((H, W))
    m = (x + y == min(H, W) - 1) if anti else (x == y)
    return np.where(m, FG, 0).astype(np.uint8)


def uniform(H: int, W: int, value: int = 255) -> np.ndarray:
    return np.full((H, W), value, dtype=np.uint8)


def frames(B: int, H: int, W: int, seed0: int = 4000, first: int = 0) -> np.ndarray:
    """Video-like batch (config C4): frame f (= first .. first+B-1) is
    texture(seed0+f) thresholded at a density cycling through 0.2..0.6."""
    dens = (0.2, 0.3, 0.4, 0.5, 0.6)
    out = np.empty((B, H, W), dtype=np.uint8)
    for i in range(B):
        f = first + i
        out[i] = texture(H, W, seed0 + f, dens[f % len(dens)], octaves=((64, 4), (16, 2), (4, 1)))
    return out


def percolation_density(connectivity: int) -> float:
    """Site-percolation thresholds of the square lattice (4: 0.5927, 8: 0.4073)."""
    return 0.5927 if connectivity == 4 else 0.4073


def _check_dims(H: int, W: int) -> None:
    if H < 1 or W < 1:
        raise ValueError(f"invalid dimensions {H}x{W}")
