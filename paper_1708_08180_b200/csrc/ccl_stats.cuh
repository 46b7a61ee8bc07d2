// ccl_stats.cuh -- per-component statistics of a canonical label map
// (SURVEY.md 8(f) NEXT-3): "the size and location of each dot" the paper's
// motivating applications need, plus the compaction of the
// labels to 1..K in label order (SPEC.md:336's renumbering op).
//
// Input: labels from ccl_label (0 = background, else 1 + the minimum raster
// index of the component).  A component's root is the pixel whose label is
// its own index + 1, so the components, in increasing label order, are the
// roots in raster order:
//   S1 count the roots of every 4096-px chunk;
//   S2 exclusive scan of the chunk counts per image (component ids);
//   S3 each root gets its id (rank) in the sparse map M[root] and initialises
//      its output record;
//   S4 every foreground pixel is counted in record M[label - 1] (and, when
//      asked, written to the relabelled map as M[label - 1] + 1): a warp walks
//      its own contiguous range of 32-px segments; within a segment, runs of
//      equal (component, row) have closed-form statistics (area = length,
//      x range, coordinate sums); the run that reaches a segment's end is
//      carried in registers into the next segment, the others accumulate in
//      a 1024-slot shared-memory hash table (linear probing, 8 probes; a full
//      neighbourhood falls back to global atomics) that the block flushes at
//      the end -- a giant component costs a few global atomics per block.
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ccl.h"

namespace ccl {
namespace stats {

constexpr int kChunk = 4096;  // pixels per S1/S3 block (256 threads x 16)
constexpr int kT = 256;
constexpr int kSlots = 1024;  // shared table (36 KB), linear probing
constexpr int kProbe = 8;     // slots tried before falling back to global atomics

__global__ void __launch_bounds__(kT) k_stats_count(const int32_t* __restrict__ labels, long long npx, int nchunks,
                                                    int32_t* __restrict__ cnt) {
    const int b = blockIdx.y, c = blockIdx.x;
    const int32_t* L = labels + size_t(b) * size_t(npx);
    const long long base = (long long)c * kChunk;
    int n = 0;
#pragma unroll 4
    for (int k = 0; k < kChunk / kT; ++k) {
        const long long i = base + k * kT + threadIdx.x;
        if (i < npx && L[i] == int(i) + 1) ++n;
    }
    n = __reduce_add_sync(0xFFFFFFFFu, unsigned(n));
    __shared__ int ws[kT / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < kT / 32; ++w) s += ws[w];
        cnt[size_t(b) * nchunks + c] = s;
    }
}

// one block per image: exclusive scan of the chunk counts, total -> counts[b]
__global__ void __launch_bounds__(1024) k_stats_scan(int32_t* __restrict__ cnt, int nchunks, int32_t* __restrict__ counts) {
    __shared__ int carry, wsum[32];
    int32_t* C = cnt + size_t(blockIdx.x) * nchunks;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < nchunks; base += 1024) {
        const int i = base + threadIdx.x;
        const int v = i < nchunks ? C[i] : 0;
        int x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            int s = wsum[lane];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, s, d);
                if (lane >= d) s += y;
            }
            wsum[lane] = s;  // inclusive over warps
        }
        __syncthreads();
        const int excl = carry + (w > 0 ? wsum[w - 1] : 0) + x - v;
        if (i < nchunks) C[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[blockIdx.x] = carry;
}

// ranks of the roots (component ids, raster = label order) -> M; output
// records initialised
__global__ void __launch_bounds__(kT) k_stats_rank(const int32_t* __restrict__ labels, long long npx, int W,
                                                   int nchunks, const int32_t* __restrict__ off,
                                                   int32_t* __restrict__ M, ccl_component_t* __restrict__ out,
                                                   long long max_components) {
    const int b = blockIdx.y, c = blockIdx.x;
    const int32_t* L = labels + size_t(b) * size_t(npx);
    int32_t* Mb = M + size_t(b) * size_t(npx);
    ccl_component_t* O = out + size_t(b) * size_t(max_components);
    const long long base = (long long)c * kChunk + (long long)threadIdx.x * (kChunk / kT);  // 16 consecutive px
    unsigned flags = 0;
    if (base + kChunk / kT <= npx && (npx & 3) == 0 && (reinterpret_cast<uintptr_t>(labels) & 15) == 0) {
        // 4 x 16-byte loads (16-B aligned: aligned base, npx % 4 == 0); else scalar
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int4 v = __ldcs(reinterpret_cast<const int4*>(L + base) + q);
            const int i0 = int(base) + 4 * q + 1;
            flags |= (unsigned(v.x == i0) | unsigned(v.y == i0 + 1) << 1 | unsigned(v.z == i0 + 2) << 2 |
                      unsigned(v.w == i0 + 3) << 3) << (4 * q);
        }
    } else {
#pragma unroll
        for (int k = 0; k < kChunk / kT; ++k) {
            const long long i = base + k;
            if (i < npx && L[i] == int(i) + 1) flags |= 1u << k;
        }
    }
    const int n = __popc(flags);
    // block exclusive scan of n
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = n;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, x, d);
        if (lane >= d) x += y;
    }
    __shared__ int wsum[kT / 32];
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int before = 0;
    for (int v = 0; v < w; ++v) before += wsum[v];
    int r = off[size_t(b) * nchunks + c] + before + x - n;
    while (flags) {
        const int k = __ffs(flags) - 1;
        flags &= flags - 1;
        const long long i = base + k;
        Mb[i] = r;
        if (r < max_components) {
            ccl_component_t e;
            e.label = int(i) + 1;
            e.area = 0;
            e.x_min = INT_MAX;
            e.y_min = INT_MAX;
            e.x_max = -1;
            e.y_max = -1;
            e.sum_x = 0;
            e.sum_y = 0;
            O[r] = e;
        }
        ++r;
    }
}

struct Acc {
    int key[kSlots];  // component id, -1 = free
    int area[kSlots], x0[kSlots], y0[kSlots], x1[kSlots], y1[kSlots];
    unsigned long long sx[kSlots], sy[kSlots];
};

__device__ __forceinline__ void add_global(ccl_component_t* e, int area, int x0, int y0, int x1, int y1,
                                           unsigned long long sx, unsigned long long sy) {
    atomicAdd(&e->area, area);
    atomicMin(&e->x_min, x0);
    atomicMin(&e->y_min, y0);
    atomicMax(&e->x_max, x1);
    atomicMax(&e->y_max, y1);
    atomicAdd(reinterpret_cast<unsigned long long*>(&e->sum_x), sx);
    atomicAdd(reinterpret_cast<unsigned long long*>(&e->sum_y), sy);
}

// every foreground pixel -> its component's record (grid-stride over pixels
// of image blockIdx.y; each block aggregates in its shared table)
__global__ void __launch_bounds__(kT) k_stats_accum(const int32_t* __restrict__ labels, long long npx, int W,
                                                    const int32_t* __restrict__ M, ccl_component_t* __restrict__ out,
                                                    long long max_components, int32_t* __restrict__ relabel) {
    __shared__ Acc a;
    const int b = blockIdx.y;
    const int32_t* L = labels + size_t(b) * size_t(npx);
    const int32_t* Mb = M + size_t(b) * size_t(npx);
    ccl_component_t* O = out + size_t(b) * size_t(max_components);
    for (int s = threadIdx.x; s < kSlots; s += kT) {
        a.key[s] = -1;
        a.area[s] = 0;
        a.x0[s] = INT_MAX;
        a.y0[s] = INT_MAX;
        a.x1[s] = -1;
        a.y1[s] = -1;
        a.sx[s] = 0;
        a.sy[s] = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    // each warp walks its own contiguous range of 32-px segments, so the
    // component of one segment usually continues into the next: that one is
    // accumulated in registers (warp-uniform) and only flushed when it ends
    const long long nseg = (npx + 31) / 32;
    const long long nwarp = (long long)gridDim.x * (kT / 32);
    const long long gw = (long long)blockIdx.x * (kT / 32) + (threadIdx.x >> 5);
    const long long per = (nseg + nwarp - 1) / nwarp;
    const long long s0 = gw * per, s1 = min(nseg, s0 + per);
    int acid = -1, aarea = 0, ax0 = 0, ay0 = 0, ax1 = 0, ay1 = 0;
    unsigned long long asx = 0, asy = 0;
    auto flush = [&](int c, int ar, int x0, int y0, int x1, int y1, unsigned long long sx, unsigned long long sy) {
        int slot = (c * 0x9E3779B1u) >> 22;  // 10-bit multiplicative hash
        int k = -2;
        for (int pr = 0; pr < kProbe; ++pr, slot = (slot + 1) & (kSlots - 1)) {
            k = a.key[slot];
            if (k == c) break;
            if (k == -1) {
                k = atomicCAS(&a.key[slot], -1, c);
                if (k == -1 || k == c) break;
            }
        }
        if (k == -1 || k == c) {
            atomicAdd(&a.area[slot], ar);
            atomicMin(&a.x0[slot], x0);
            atomicMin(&a.y0[slot], y0);
            atomicMax(&a.x1[slot], x1);
            atomicMax(&a.y1[slot], y1);
            atomicAdd(&a.sx[slot], sx);
            atomicAdd(&a.sy[slot], sy);
        } else {
            add_global(O + c, ar, x0, y0, x1, y1, sx, sy);
        }
    };
    // coordinates of the segment's first pixel, advanced without divisions
    int sy0 = 0, sx0 = 0;
    if (s0 < s1) {
        const unsigned i0 = unsigned(s0 * 32);
        sy0 = int(i0 / unsigned(W));
        sx0 = int(i0 - unsigned(sy0) * unsigned(W));
    }
    constexpr int U = 8;  // segments whose loads are in flight together
    for (long long sb = s0; sb < s1; sb += U) {
        int lv[U], cv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = (sb + u) * 32 + lane;
            lv[u] = (sb + u < s1 && i < npx) ? __ldcs(L + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) cv[u] = lv[u] > 0 ? __ldg(Mb + lv[u] - 1) : -1;
        if (relabel) {  // the compact numbering 1..K: component id + 1, background 0
            int32_t* Rb = relabel + size_t(b) * size_t(npx);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long i = (sb + u) * 32 + lane;
                if (sb + u < s1 && i < npx) __stcs(Rb + i, cv[u] + 1);
            }
        }
        // one loop body for the U segments (a fully unrolled body thrashed the
        // instruction cache: 30 % of the stall samples); cv[] rotates so that
        // every index stays static
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
        if (sb + u >= s1) break;
        int cid = cv[0], x = sx0 + lane, y = sy0;
#pragma unroll
        for (int k = 0; k + 1 < U; ++k) cv[k] = cv[k + 1];
        if (cid >= max_components) cid = -1;
        while (x >= W) {  // once per row crossing (W >= 32), more often for narrow images
            x -= W;
            ++y;
        }
        sx0 += 32;
        while (sx0 >= W) {
            sx0 -= W;
            ++sy0;
        }
        // fast paths: an all-background segment, and a segment lying wholly in
        // one row of the component carried in registers
        const unsigned bgm = __ballot_sync(0xFFFFFFFFu, cid < 0);
        if (bgm == 0xFFFFFFFFu) continue;
        const int y_first = __shfl_sync(0xFFFFFFFFu, y, 0), x_first = __shfl_sync(0xFFFFFFFFu, x, 0);
        if (acid >= 0 && __all_sync(0xFFFFFFFFu, cid == acid && y == y_first)) {
            aarea += 32;
            ax0 = min(ax0, x_first);
            ax1 = max(ax1, x_first + 31);
            ay0 = min(ay0, y_first);
            ay1 = max(ay1, y_first);
            asx += 32ull * unsigned(x_first) + 496ull;
            asy += 32ull * unsigned(y_first);
            continue;
        }
        // runs of equal (component, row) along the segment: every statistic
        // of a run is a closed form of its first x and its length
        const int pc = __shfl_up_sync(0xFFFFFFFFu, cid, 1), py = __shfl_up_sync(0xFFFFFFFFu, y, 1);
        const unsigned brk = __ballot_sync(0xFFFFFFFFu, lane == 0 || cid != pc || y != py);
        const unsigned above = brk & ~((2u << lane) - 1u);  // breaks after this lane (lane 31: none)
        const int len = (lane == 31 ? 32 : (above ? __ffs(above) - 1 : 32)) - lane;  // valid at run starts
        const bool start = cid >= 0 && ((brk >> lane) & 1u);
        const int area = len;
        const int x0 = x, x1 = x + len - 1, y0 = y, y1 = y;
        const unsigned long long sx = (unsigned long long)len * unsigned(x) + (unsigned long long)(len * (len - 1) / 2);
        const unsigned long long sy = (unsigned long long)len * unsigned(y);
        const int first_cid = __shfl_sync(0xFFFFFFFFu, cid, 0);
        const int lastL = 31 - __clz(brk);                  // start lane of the run holding lane 31
        const int last_cid = __shfl_sync(0xFFFFFFFFu, cid, 31);
        // the register accumulator continues with the segment's first run if it
        // is the same component, else it is flushed
        bool merged_first = false;
        if (acid >= 0 && first_cid == acid) {
            aarea += __shfl_sync(0xFFFFFFFFu, area, 0);
            ax0 = min(ax0, __shfl_sync(0xFFFFFFFFu, x0, 0));
            ax1 = max(ax1, __shfl_sync(0xFFFFFFFFu, x1, 0));
            ay0 = min(ay0, __shfl_sync(0xFFFFFFFFu, y0, 0));
            ay1 = max(ay1, __shfl_sync(0xFFFFFFFFu, y1, 0));
            asx += __shfl_sync(0xFFFFFFFFu, sx, 0);
            asy += __shfl_sync(0xFFFFFFFFu, sy, 0);
            merged_first = true;
        } else {
            if (acid >= 0 && lane == 0) flush(acid, aarea, ax0, ay0, ax1, ay1, asx, asy);
            acid = -1;
        }
        // ... and then holds the run that reaches the segment's end
        const bool last_is_first = lastL == 0;
        if (last_cid >= 0 && !(last_is_first && merged_first)) {
            if (acid >= 0 && lane == 0) flush(acid, aarea, ax0, ay0, ax1, ay1, asx, asy);
            acid = last_cid;
            aarea = __shfl_sync(0xFFFFFFFFu, area, lastL);
            ax0 = __shfl_sync(0xFFFFFFFFu, x0, lastL);
            ax1 = __shfl_sync(0xFFFFFFFFu, x1, lastL);
            ay0 = __shfl_sync(0xFFFFFFFFu, y0, lastL);
            ay1 = __shfl_sync(0xFFFFFFFFu, y1, lastL);
            asx = __shfl_sync(0xFFFFFFFFu, sx, lastL);
            asy = __shfl_sync(0xFFFFFFFFu, sy, lastL);
        }
        // every other run: its first lane flushes it
        const bool held = (lane == 0 && merged_first) || (lane == lastL && last_cid >= 0);
        if (start && !held) flush(cid, area, x0, y0, x1, y1, sx, sy);
        }
    }
    if (acid >= 0 && lane == 0) flush(acid, aarea, ax0, ay0, ax1, ay1, asx, asy);
    __syncthreads();
    for (int s = threadIdx.x; s < kSlots; s += kT)
        if (a.key[s] >= 0) add_global(O + a.key[s], a.area[s], a.x0[s], a.y0[s], a.x1[s], a.y1[s], a.sx[s], a.sy[s]);
}

}  // namespace stats
}  // namespace ccl
