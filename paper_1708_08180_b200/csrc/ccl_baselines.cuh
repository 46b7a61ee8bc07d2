// ccl_baselines.cuh -- the paper's three comparison methods on sm_100a
// (Table 2), written
// plainly at pixel granularity in the thread-block shapes the paper ran them
// with ({32,16,1} for LE and conventional UF, {512,1,1} for
// line-based UF).  They exist to measure the paper's relative claims on B200
// (ours vs UF ~3.4x at 4096^2, vs line UF ~1.3x, vs LE), not
// as product paths.  All produce the same canonical labels as the main path
// (0 = background, else 1 + minimum raster index of the component): every
// union links the larger root under the smaller (min-root), and LE propagates
// minimum labels, so each component converges to its minimum index.
//
//  * UF (conventional parallel union-find, [oliveira2010study], PAPER.md:37,
//    68-70): local merge -- per-pixel union-find in shared memory over a
//    32x16 block (no coarse labeling), each pixel's local root converted to a
//    global index; global merge -- one thread per pixel on a tile-boundary
//    row/column unions every crossing edge in global memory; link -- every
//    pixel flattened to its root.
//  * Line UF ([yonehara2015line]): local merge along 512-px
//    row segments (one block each), then a global union over ALL cells (every
//    pixel with its upper neighbours and the segment-boundary left neighbour),
//    then link.
//  * LE (label equivalence, [CCLinCUDA] / [hawick2010parallel], PAPER.md:35,
//    400): multi-pass -- scan (each pixel's minimum neighbour label recorded
//    as an equivalence of its current label), analysis (labels resolved
//    through the equivalence chains), relabel; repeated until a scan changes
//    nothing (one device->host flag read per iteration, as that method does).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ccl {
namespace base {

constexpr int kBX = 32, kBY = 16;  // {32,16,1} blocks
constexpr int kLine = 512;         // {512,1,1} blocks

// min-root union in a parent array (shared or global) of indices
__device__ __forceinline__ int find_root(const volatile int32_t* P, int a) {
    int p = P[a];
    while (p != a) {
        a = p;
        p = P[a];
    }
    return a;
}

// find with path splitting (each visited node re-pointed at its grandparent;
// only ancestors are written, so concurrent finds stay valid) -- keeps the
// global forests shallow, as the comparison methods' own implementations do
__device__ __forceinline__ int find_split(volatile int32_t* P, int a) {
    int p = P[a];
    while (p != a) {
        const int gp = P[p];
        if (gp != p) P[a] = gp;
        a = p;
        p = gp;
    }
    return a;
}

__device__ __forceinline__ void union_min(int32_t* P, int a, int b) {
    volatile int32_t* V = P;
    while (true) {
        a = find_split(V, a);
        b = find_split(V, b);
        if (a == b) return;
        if (a < b) { int t = a; a = b; b = t; }
        const int old = atomicMin(P + a, b);
        if (old == a) return;
        a = old;
    }
}

__device__ __forceinline__ bool fg_at(const uint8_t* im, int W, int H, int x, int y) {
    return x >= 0 && x < W && y >= 0 && y < H && im[size_t(y) * W + x] != 0;
}

// ---------------------------------------------------------------- UF (2D)
// Local merge: G[p] = global index of p's local root (fg), -1 (bg).
// EQ (equal-value mode, NEXT-2): every in-image pixel takes part and two
// neighbours are connected iff their values are equal (the paper's raw
// comparisons dBuff[tid] == dBuff[tid-1]); else foreground
// (nonzero) pixels, connected iff both are foreground.
template <bool EQ>
__device__ __forceinline__ bool linked(const uint8_t* im, int W, int H, int x, int y, int xx, int yy) {
    if (xx < 0 || xx >= W || yy < 0 || yy >= H) return false;
    const uint8_t a = im[size_t(y) * W + x], c = im[size_t(yy) * W + xx];
    return EQ ? a == c : (a != 0 && c != 0);
}

template <int CONN, bool EQ = false>
__global__ void __launch_bounds__(kBX * kBY) k_uf_local(const uint8_t* __restrict__ img, int H, int W,
                                                        long long npx, int32_t* __restrict__ G) {
    __shared__ int32_t P[kBX * kBY];
    __shared__ uint8_t F[kBX * kBY];  // pixel value (EQ) / foreground flag
    const int b = blockIdx.z;
    const uint8_t* im = img + size_t(b) * size_t(npx);
    int32_t* Gb = G + size_t(b) * size_t(npx);
    const int lx = threadIdx.x, ly = threadIdx.y, tid = ly * kBX + lx;
    const int x = blockIdx.x * kBX + lx, y = blockIdx.y * kBY + ly;
    const bool inside = x < W && y < H;
    const uint8_t v = inside ? im[size_t(y) * W + x] : 0;
    const bool f = EQ ? inside : v != 0;
    P[tid] = tid;
    F[tid] = EQ ? v : uint8_t(f);
    __syncthreads();
    if (f) {
        // in-tile neighbours (W, N, NW are inside the image whenever this
        // pixel is; NE is checked): EQ compares values, else both foreground
        auto m = [&](int t2) { return EQ ? F[t2] == v : F[t2] != 0; };
        if (lx > 0 && m(tid - 1)) union_min(P, tid, tid - 1);
        if (ly > 0 && m(tid - kBX)) union_min(P, tid, tid - kBX);
        if (CONN == 8 && ly > 0 && lx > 0 && m(tid - kBX - 1)) union_min(P, tid, tid - kBX - 1);
        if (CONN == 8 && ly > 0 && lx + 1 < kBX && x + 1 < W && m(tid - kBX + 1)) union_min(P, tid, tid - kBX + 1);
    }
    __syncthreads();
    if (x < W && y < H) {
        int v = -1;
        if (f) {
            const int r = find_root(P, tid);  // l_x = r mod 32, l_y = r div 32 (reading R7)
            v = (blockIdx.y * kBY + r / kBX) * W + blockIdx.x * kBX + r % kBX;
        }
        Gb[size_t(y) * W + x] = v;
    }
}

// Global merge: one thread per pixel on a tile-boundary line; unions every
// backward edge (W, NW, N, NE) of that pixel that crosses a tile boundary
// (reading R10).  Pixel set: rows y % 16 == 0 (y > 0), then columns
// x % 32 == 0 (x > 0) and x % 32 == 31 (x + 1 < W: the NE edge's tile
// crossing), rows excluded from the column part to count each pixel once.
template <int CONN, bool EQ = false>
__global__ void k_uf_global(const uint8_t* __restrict__ img, int H, int W, long long npx, int32_t* __restrict__ G,
                            int nrows, int ncols, long long per_img) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (i >= per_img) return;
    int x, y;
    const long long nr = (long long)nrows * W;
    if (i < nr) {
        y = int(i / W + 1) * kBY;
        x = int(i % W);
    } else {
        const long long j = i - nr;
        const int c = int(j / H);
        y = int(j % H);
        x = (c >> 1) * kBX + ((c & 1) ? kBX - 1 : kBX);  // c even: x = 32k (k >= 1); odd: x = 32k + 31
        if (x >= W || (y % kBY == 0 && y > 0)) return;
    }
    const uint8_t* im = img + size_t(b) * size_t(npx);
    int32_t* Gb = G + size_t(b) * size_t(npx);
    if (!EQ && !fg_at(im, W, H, x, y)) return;
    const int p = y * W + x;
    const bool xb = x % kBX == 0, yb = y % kBY == 0, xe = (x + 1) % kBX == 0;
    if (xb && linked<EQ>(im, W, H, x, y, x - 1, y)) union_min(Gb, Gb[p], Gb[p - 1]);
    if (yb && linked<EQ>(im, W, H, x, y, x, y - 1)) union_min(Gb, Gb[p], Gb[p - W]);
    if (CONN == 8) {
        if ((xb || yb) && linked<EQ>(im, W, H, x, y, x - 1, y - 1)) union_min(Gb, Gb[p], Gb[p - W - 1]);
        if ((xe || yb) && linked<EQ>(im, W, H, x, y, x + 1, y - 1)) union_min(Gb, Gb[p], Gb[p - W + 1]);
    }
}

// Link: labels_out[p] = off + root (fg; off = 1, or 0 in equal-value mode)
// or 0 (background, binary mode only).
__global__ void k_link_flat(const int32_t* __restrict__ G, int32_t* __restrict__ out, long long n, long long npx,
                            int off = 1) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long b = i / npx;
        const int32_t* Gb = G + b * npx;
        const int v = G[i];
        out[i] = v < 0 ? 0 : find_root(Gb, v) + off;
    }
}

// ------------------------------------------------------------ line UF
// Local merge along a 512-px row segment: G[p] = global index of the first
// pixel of p's run within the segment (fg), -1 (bg).
__global__ void __launch_bounds__(kLine) k_line_local(const uint8_t* __restrict__ img, int H, int W, long long npx,
                                                      int32_t* __restrict__ G) {
    __shared__ int32_t P[kLine];
    __shared__ uint8_t F[kLine];
    const int b = blockIdx.z, y = blockIdx.y, x = blockIdx.x * kLine + threadIdx.x, t = threadIdx.x;
    const uint8_t* im = img + size_t(b) * size_t(npx);
    const bool f = fg_at(im, W, H, x, y);
    P[t] = t;
    F[t] = f;
    __syncthreads();
    if (f && t > 0 && F[t - 1]) union_min(P, t, t - 1);
    __syncthreads();
    if (x < W) G[size_t(b) * size_t(npx) + size_t(y) * W + x] = f ? y * W + blockIdx.x * kLine + find_root(P, t) : -1;
}

// Global merge over ALL cells: upper neighbours (N; NW, NE for 8-conn) and
// the left neighbour across a segment boundary.
template <int CONN>
__global__ void k_line_global(const uint8_t* __restrict__ img, int H, int W, long long npx, int32_t* __restrict__ G) {
    const int b = blockIdx.z, y = blockIdx.y, x = blockIdx.x * kLine + threadIdx.x;
    const uint8_t* im = img + size_t(b) * size_t(npx);
    if (!fg_at(im, W, H, x, y)) return;
    int32_t* Gb = G + size_t(b) * size_t(npx);
    const int p = y * W + x;
    if (x % kLine == 0 && fg_at(im, W, H, x - 1, y)) union_min(Gb, Gb[p], Gb[p - 1]);
    if (fg_at(im, W, H, x, y - 1)) union_min(Gb, Gb[p], Gb[p - W]);
    if (CONN == 8) {
        if (fg_at(im, W, H, x - 1, y - 1)) union_min(Gb, Gb[p], Gb[p - W - 1]);
        if (fg_at(im, W, H, x + 1, y - 1)) union_min(Gb, Gb[p], Gb[p - W + 1]);
    }
}

// ------------------------------------------------------------------ LE
__global__ void k_le_init(const uint8_t* __restrict__ img, int32_t* __restrict__ L, int32_t* __restrict__ R,
                          long long n, long long npx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int v = img[i] ? int(i % npx) : -1;
        L[i] = v;
        R[i] = v;
    }
}

// Scan: the minimum label among p and its fg neighbours; if smaller than
// p's label, record the equivalence R[L[p]] <- min (atomicMin) and flag.
template <int CONN>
__global__ void __launch_bounds__(kBX * kBY) k_le_scan(const int32_t* __restrict__ L, int32_t* __restrict__ R, int H,
                                                       int W, long long npx, int* __restrict__ changed) {
    const int b = blockIdx.z;
    const int x = blockIdx.x * kBX + threadIdx.x, y = blockIdx.y * kBY + threadIdx.y;
    if (x >= W || y >= H) return;
    const int32_t* Lb = L + size_t(b) * size_t(npx);
    const int l = Lb[size_t(y) * W + x];
    if (l < 0) return;
    int m = l;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            if ((dx == 0 && dy == 0) || (CONN == 4 && dx != 0 && dy != 0)) continue;
            const int xx = x + dx, yy = y + dy;
            if (xx < 0 || xx >= W || yy < 0 || yy >= H) continue;
            const int v = Lb[size_t(yy) * W + xx];
            if (v >= 0 && v < m) m = v;
        }
    if (m < l) {
        atomicMin(R + size_t(b) * size_t(npx) + l, m);
        *changed = 1;
    }
}

// Analysis: every label root follows its equivalence chain to the end.
__global__ void k_le_analysis(const int32_t* __restrict__ L, int32_t* __restrict__ R, long long n, long long npx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long b = i / npx;
        const int l = L[i];
        if (l != int(i % npx)) continue;  // only label owners
        volatile int32_t* Rb = R + b * npx;
        int r = Rb[l];  // R[x] <= x: the chain ends at a fixed point
        while (true) {
            const int rr = Rb[r];
            if (rr == r) break;
            r = rr;
        }
        Rb[l] = r;
    }
}

// Relabel: L[p] <- R[L[p]].
__global__ void k_le_relabel(int32_t* __restrict__ L, const int32_t* __restrict__ R, long long n, long long npx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int l = L[i];
        if (l >= 0) L[i] = R[(i / npx) * npx + l];
    }
}

__global__ void k_le_out(const int32_t* __restrict__ L, int32_t* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = L[i] + 1;  // -1 (bg) -> 0
}

}  // namespace base
}  // namespace ccl
