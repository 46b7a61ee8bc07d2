// ccl_kernels.cuh -- sm_100a kernels of the three-phase block-parallel union-find
// CCL of arxiv 1708.08180:
//   K1 k_local_merge  "Local UF merge with coarse labeling"  (Alg. 1)
//   K2 k_boundary     "Boundary analysis"                    (Alg. 2)
//   K3 k_link         "Final link"                           (§2.3)
//
// B200 design:
//  * A tile is TY rows x 1024 px; one warp owns a 1024-px tile row, lane l the
//    32-px mask word l.  The image is read once with coalesced 128-bit loads and
//    turned into foreground bit masks (fg = byte != 0, reading R1).
//  * Coarse labeling (Alg. 1 l.9-24: row scan + column scan + row-column
//    unification) becomes exact row-run detection on the masks: a run start is
//    m & ~(m<<1 | carry); every pixel's provisional label is its run's start
//    (the lowest equivalent label in its row).
//  * Local UF (Alg. 1 l.25-33) unions runs of adjacent rows only at the START
//    of each overlap segment (4-conn) plus the NE/NW diagonal run contacts
//    (8-conn): one union per adjacent run pair instead of one per pixel edge.
//    The parent array lives in shared memory, indexed by (tile-local index>>1)
//    (two run starts are never horizontally adjacent), min-root atomicMin union.
//  * Local->global index conversion (Alg. 1 l.34-39) uses
//    g = (y0 + l/1024)*W + x0 + l%1024 (reading R7: l_x = l mod T_x).
//  * K1 writes only (a) the bit-packed mask (1/8 B/px) and (b) for tile-EDGE
//    pixels, the global index of their local root into the global parent array
//    G (workspace), plus G[root] = root.  No per-pixel label map is written.
//  * K2 runs lock-free min-root union (atomicMin retry, reading R11) in G over
//    every foreground edge crossing a tile boundary (reading R9/R10).
//  * K3 re-derives the local labels from the bit mask (deterministic: the same
//    roots), resolves edge-touching roots through G, and streams 1 + root (or 0)
//    for every pixel with 128-bit evict-first stores.  DRAM traffic per pixel
//    ~ 1 B (image) + 4 B (labels) + 1/4 B (mask) + edge entries.
#pragma once
#include <cassert>
#include <cstdio>
#include <climits>
#include <cstdint>
#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded on the host in ccl_api.cu)
#include <cuda_runtime.h>

#ifdef CCL_CHECK
#define CCL_ASSERT(c) assert(c)
#define CCL_LOOP_GUARD(name) int name##_guard = 0
#define CCL_LOOP_TICK(name) assert(++name##_guard < (1 << 22))
#else
#define CCL_ASSERT(c) ((void)0)
#define CCL_LOOP_GUARD(name) ((void)0)
#define CCL_LOOP_TICK(name) ((void)0)
#endif

namespace ccl {

constexpr int kTileW = 1024;   // pixels per tile row
constexpr int kWords = 32;     // 32-bit mask words per tile row
constexpr int kThreads = 256;  // threads per K1/K3 block
constexpr int kWarps = kThreads / 32;
// K1 block size: 256 threads for 8- and 16-row tiles (5 blocks per SM); for
// 32-row tiles 512 threads (16 warps, two rows each: the same register
// prefetch of the next tile as 16-row tiles) and 2 blocks per SM, whose
// 110 KB of shared memory hold the run lists of an i.i.d.-noise tile
// (~8192 runs) instead of sending it to the global scratch path.
#ifndef CCL_K1_T32
#define CCL_K1_T32 256  // 512 measured: texture K1 49.7 -> 53.9 us, noise 2.0 -> 0.8 ms (profiles/r02_ab_k1_ty32_256_vs_512.txt)
#endif
template <int TY>
__host__ __device__ constexpr int k1_threads() { return TY > 16 ? CCL_K1_T32 : 256; }
template <int TY>
__host__ __device__ constexpr int k1_warps() { return k1_threads<TY>() / 32; }

// Run lists of a tile live in shared memory up to k1_cap runs (natural
// images: a few hundred; i.i.d. noise at density 1/2: ~4096 per 16 rows),
// which keeps the block at 45 KB -- with one prefetch register set (44
// registers) 5 blocks (40 warps) per SM; measured: 4 blocks 46.8 us, 5 blocks
// 43.6 us on C3 texture.  A tile with more runs (noise in 32-row tiles,
// period-2 stripes, checkerboards: up to TY*512) is labelled in maximal row
// ranges that fit (k1_range), whose boundaries are unioned like tile
// boundaries.
#ifndef CCL_K1_CAP16
#define CCL_K1_CAP16 4576
#endif
#ifndef CCL_K1_BLOCKS
#define CCL_K1_BLOCKS 5
#endif
#ifndef CCL_K1_BLOCKS32
#define CCL_K1_BLOCKS32 5  // 32-row tiles: 5 blocks per SM (48 registers; 3456 runs in shared memory)
#endif
__host__ __device__ constexpr int k1_cap32() {
    // 16 KB of row words; 512 threads: 11776 runs (110 KB, 2 blocks per SM);
    // 256 threads: 4800 runs at 4 blocks per SM (54 KB), 3456 at 5 (44 KB),
    // 2400 at 6 (36 KB).  Measured (C3, 32-row tiles, µs/step): 6 vs 5 blocks
    // texture 103.1 vs 103.3, C4 3190 vs 3242, noise 694 vs 734, percolation
    // 673 vs 675, but the smaller cap raises the worst-case edge slots per
    // tile (9 row ranges instead of 6): workspace 4.5 instead of 3.7 B/px;
    // 4 blocks: texture 105.4.  5 kept.
#ifdef CCL_K1_CAP32
    return CCL_K1_CAP32;
#else
    return CCL_K1_T32 == 512 ? 11776 : (CCL_K1_BLOCKS32 == 4 ? 4800 : (CCL_K1_BLOCKS32 == 6 ? 2400 : 3456));
#endif
}
__host__ __device__ constexpr int k1_cap_n(int TY) {
    return TY * kTileW / 2 < (TY > 16 ? k1_cap32() : CCL_K1_CAP16) ? TY * kTileW / 2
                                                                   : (TY > 16 ? k1_cap32() : CCL_K1_CAP16);
}
template <int TY>
__host__ __device__ constexpr int k1_cap() { return k1_cap_n(TY); }
// most row ranges a tile can need: every range but the last holds more than
// k1_cap - 512 runs (else one more row would have fitted)
__host__ __device__ constexpr int k1_max_ranges(int TY) {
    return TY * kTileW / 2 <= k1_cap_n(TY) ? 1 : 1 + (TY * kTileW / 2) / (k1_cap_n(TY) - kTileW / 2 + 1);
}
#ifndef CCL_K2_WARPS
#define CCL_K2_WARPS 8  // warps (boundary tasks) per K2 block
#endif
constexpr int kK2Warps = CCL_K2_WARPS;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kTag = int(0x80000000u);

// Division by a runtime-invariant divisor d >= 1 for numerators n < 2^31 via
// a precomputed multiplier (Granlund-Montgomery): q = (umulhi(n, mul) + n) >> shr.
struct FastDiv {
    unsigned d, mul, shr;
    __host__ __device__ FastDiv() : d(1), mul(0), shr(0) {}
    __host__ explicit FastDiv(unsigned dd) : d(dd) {
        shr = 0;
        while ((1ull << shr) < dd) ++shr;
        mul = unsigned(((1ull << 32) * ((1ull << shr) - dd)) / dd + 1);
    }
    __device__ __forceinline__ unsigned div(unsigned n) const { return (__umulhi(n, mul) + n) >> shr; }
};

struct Geom {
    int B, H, W;       // batch, rows, columns
    int WW;            // mask words per image row = ceil(W/32)
    int tiles_x;       // ceil(W/1024)
    int tiles_y;       // ceil(H/TY)
    long long npx;     // H*W  (per image)
    long long nwords;  // H*WW (per image)
    FastDiv div_tx, div_ty;  // by tiles_x, tiles_y
    FastDiv div_ty1, div_tx1, div_vg;  // K2 task decode: tiles_y - 1, tiles_x - 1, vertical task groups
    // strip mode (row-strip sharding of one image over several GPUs):
    int label_off;     // added to every label (row0 * W_total: labels are global)
    int force_top;     // the image's first row borders another strip
    int force_bottom;  // the image's last row borders another strip
    // foreground test fused into K1's load (ccl_label_threshold_async):
    // value >= thr; thr_k = the SWAR constant of nzc4 (K1 template THR 1 / 2)
    int thr;
    uint32_t thr_k;
    int k3_early;      // K3 may read K1's outputs before its PDL wait (K1 finished before K3's predecessor)
    unsigned ntiles;   // tiles of the whole batch: the stride of the edge-slot numbering
    int strip;         // strip mode (row-strip sharding): K1 also clears the strip marks F of its edge slots
    // K1 -> K2 overlap (both in one call): K1 publishes each finished tile as
    // ready[t] = epoch (unique per call) and lets K2 launch early; K2's tasks
    // wait for their tiles' flags instead of for K1's completion.  0: off.
    unsigned long long epoch;
    unsigned long long* ready;
    int32_t* defer;    // K1's per-block lists of run-dense tiles (ntiles ints)
};

// One 32-px mask word with its row-run description (one 128-bit smem load).
struct __align__(16) Word {
    uint32_t m;  // foreground mask
    uint32_t s;  // run-start mask (tile-local runs)
    int32_t c;   // x (0..1023) of the run start owning bit 0 of the word (if fg), else -1
    int32_t pad;
};

// Per-run record written by K1 and read by K3 (uint32 per run, runs of a tile
// in raster order of their starts): bits 0..14 = tile-local index of the run's
// local root (row*1024 + x of its start); bits 16..31 = 1 + the root's index in
// the tile's edge-root list if its component touches a tile edge (its final
// label then comes from the boundary analysis), else 0.
#ifndef CCL_K3_RUNCACHE
#define CCL_K3_RUNCACHE 256
#endif
constexpr int kRunCache = CCL_K3_RUNCACHE;  // run records K3 prefetches per tile (128 per warp, warps 0..)
constexpr int kRL = 32;         // run records of each boundary row K1 copies into the edge brief
template <int TY>
__host__ __device__ constexpr int runs_per_tile_cap() { return TY * kTileW / 2; }
// Edge slots (the boundary analysis' union-find nodes): the i-th edge-touching
// local root of tile t (i < its edge count n) is slot i * ntiles + t -- slot
// numbers are "edge index major", so the few slots a natural image uses per
// tile (i < ~30) are packed into a few MB instead of being scattered over a
// raster-indexed H*W array (K2's dependent loads cost ~4x when they touch
// hundreds of 2 MB pages: profiles/r02_latency_sparse_pages.txt).  Slot s's
// 64-bit entry G[s] = (X << 32) | parent slot, X = the parent's image-local
// raster index (a root: its own), so the minimum-raster-index root policy
// (reading R11) is an unsigned 64-bit atomicMin.
// Within that order a 128-byte line holds 16 consecutive edge indices of ONE
// tile (line q of tile t holds i = 16q .. 16q+15), so no two tiles' entries
// share a line or sector (a layout with one tile per 8-byte step measured
// K2 25 -> 37 us: atomics and pointer-jumping stores of different tiles on
// one line), and K1 writes each tile's entries as whole 32-byte sectors.
// (capacity: every row next to a tile edge or a range boundary can carry 512
// edge roots, the columns 2 * TY, each range pads to a whole sector)
__host__ __device__ constexpr int edge_slots(int TY) {
    return (2 * k1_max_ranges(TY) * (kTileW / 2) + 2 * TY + 4 * k1_max_ranges(TY) + 15) / 16 * 16;
}
__host__ __device__ inline unsigned edge_slot(unsigned ntiles, int i, unsigned t) {
    return ((unsigned(i) >> 4) * ntiles + t) * 16u + (unsigned(i) & 15u);
}

// Per-tile edge brief E[t] (kEdgeCap ints), written by K1:
//   [0] n = number of edge-touching local roots; [1] run id of the first run
//   of the tile's last row; [kEdgeLC + r] / [kEdgeRC + r] = slot of the local
//   root of pixel (r, 0) / (r, 1023), or -1; [kEdgeR0 + i] / [kEdgeRL + i], i
//   < 32 = the run records of the first 32 runs of the first / last row (the
//   boundary analysis reads them in its first round trip).
constexpr int kEdgeLC = 2;
constexpr int kEdgeRC = 34;
constexpr int kEdgeR0 = 66;
constexpr int kEdgeRL = 98;
constexpr int kEdgeCap = 136;

// ------------------------------------------------------------------ helpers
// 4-bit mask of the nonzero bytes of w: the carry trick puts byte i's "nonzero"
// bit at bit 8i+7; one multiply by 2^21+2^14+2^7+1 moves it to bit 28+i (the
// 16 partial products land on distinct bits, so no carries) and >> 28 keeps
// the nibble.
__device__ __forceinline__ uint32_t nz4(uint32_t w) {
    const uint32_t t = (((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u;
    return (t * 0x00204081u) >> 28;
}

__device__ __forceinline__ uint32_t nz16(uint4 v) {
    uint32_t r = nz4(v.w);
    r = (r << 4) + nz4(v.z);
    r = (r << 4) + nz4(v.y);
    return (r << 4) + nz4(v.x);
}

// Thresholded variant (value >= c, SPEC.md:50-58 binarize): for c <= 128 a
// byte b passes iff (b & 0x7F) + (128 - c) reaches bit 7 or b >= 128 (THR 1,
// k = (128 - c) x 0x01010101; c = 1 is nz4); for c > 128 iff b >= 128 and
// (b & 0x7F) + (256 - c) reaches bit 7 (THR 2, k = (256 - c) x 0x01010101).
// No carry crosses a byte (each sum < 256).
template <int THR>
__device__ __forceinline__ uint32_t nzc4(uint32_t w, uint32_t k) {
    const uint32_t x = (w & 0x7F7F7F7Fu) + k;
    const uint32_t t = (THR == 2 ? (x & w) : (x | w)) & 0x80808080u;
    return (t * 0x00204081u) >> 28;
}
template <int THR>
__device__ __forceinline__ uint32_t nzc16(uint4 v, uint32_t k) {
    if (THR == 0) return nz16(v);
    uint32_t r = nzc4<THR>(v.w, k);
    r = (r << 4) + nzc4<THR>(v.z, k);
    r = (r << 4) + nzc4<THR>(v.y, k);
    return (r << 4) + nzc4<THR>(v.x, k);
}

// Programmatic dependent launch (K2, resolve and K3 are launched with the
// stream-serialisation attribute): a dependent grid is scheduled while its
// predecessor drains (C3: 151 -> 145 us/step); wait blocks until the
// predecessor has completed and its writes are visible (a no-op for a normal
// launch).  No early launch_dependents trigger: letting the next grid's
// blocks become resident before the predecessor's last blocks exit measured
// slower (K3's blocks then hold shared memory the resolve / boundary blocks
// need; 173 us with triggers at kernel entry, 148 with one in resolve).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
#ifndef CCL_K2_POLL_NS
#define CCL_K2_POLL_NS 32  // (C3 texture 99.77 vs 99.93 us at 128, 100.14 at 512; C4 and noise unchanged)
#endif
// K2 side of the K1 -> K2 overlap: one lane waits for tile t's ready flag
// (acquire), the warp synchronises behind it.
__device__ __forceinline__ void wait_tile_ready(const Geom& g, size_t t) {
    CCL_LOOP_GUARD(wr);
    while (ld_acquire_u64(g.ready + t) != g.epoch) {
        CCL_LOOP_TICK(wr);
        __nanosleep(CCL_K2_POLL_NS);
    }
}
// K3's barrier over its 256 compute threads (named barrier 1; the helper warp never joins)
__device__ __forceinline__ void k3_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory"); }

// Read-once image loads (no L1 allocation).  An L2 evict-first cache policy
// on these loads measured slower for K1 and did not help K2 (profiles r01).
__device__ __forceinline__ uint4 ld_stream_u4(const uint8_t* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ void st_stream_i4(int32_t* p, int a, int b, int c, int d) {
    asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

// K1's outputs (bit mask, run records, edge blocks, parent sectors) are stored
// with an L2 evict_last hint: the boundary analysis and K3 read them back
// right after K1, and without the hint most of them were already evicted
// again by K1's own 64 MiB image stream (ncu, cache control off: K2 / resolve
// L2 read hit rates 25 % / 21 %, K1 writing its 12.5 MB back to DRAM).
#ifndef CCL_K1_KEEP
#define CCL_K1_KEEP 1
#endif
__device__ __forceinline__ uint64_t l2_keep_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void l2_discard(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
template <typename T>
__device__ __forceinline__ void st_keep(T* p, T v) {
    static_assert(sizeof(T) == 4, "32-bit stores");
#if CCL_K1_KEEP
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(*reinterpret_cast<uint32_t*>(&v)),
                 "l"(l2_keep_policy())
                 : "memory");
#else
    *p = v;
#endif
}
__device__ __forceinline__ void st_keep_u64(uint64_t* p, uint64_t v) {
#if CCL_K1_KEEP
    asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(l2_keep_policy()) : "memory");
#else
    *p = v;
#endif
}
__device__ __forceinline__ void st_keep_v4(int4* p, int4 v) {
#if CCL_K1_KEEP
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w), "l"(l2_keep_policy())
                 : "memory");
#else
    *p = v;
#endif
}

__device__ __forceinline__ int ld_volatile(const int32_t* p) {
    return *reinterpret_cast<const volatile int32_t*>(p);
}

// x (0..1023) of the start of the tile-local run containing foreground pixel x
// of a tile row described by start masks s[] and carries c[].
__device__ __forceinline__ int run_start_x(const Word* row, int x) {
    const int w = x >> 5, bit = x & 31;
    const uint32_t below = row[w].s & (kFull >> (31 - bit));
    return below ? ((w << 5) + 31 - __clz(below)) : row[w].c;
}

// Row-run analysis of one 1024-px tile row held one word per lane: start mask
// and carry (x of the run start owning bit 0) for this lane's word.
__device__ __forceinline__ void row_runs(uint32_t m, int lane, uint32_t& s, int& c) {
    uint32_t pm = __shfl_up_sync(kFull, m, 1);
    if (lane == 0) pm = 0;
    s = m & ~((m << 1) | (pm >> 31));
    int ls = s ? ((lane << 5) + 31 - __clz(s)) : -1;  // last start in this word
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int t = __shfl_up_sync(kFull, ls, d);
        if (lane >= d) ls = max(ls, t);
    }
    int excl = __shfl_up_sync(kFull, ls, 1);
    if (lane == 0) excl = -1;
    c = (m & 1u) ? ((s & 1u) ? (lane << 5) : excl) : -1;
}

// -------------------------------------------------- global union-find (K2)
__device__ __forceinline__ void st_volatile(int32_t* p, int v) {
    *reinterpret_cast<volatile int32_t*>(p) = v;
}

#ifdef CCL_STATS
__device__ unsigned long long g_stat_unions = 0, g_stat_steps = 0, g_stat_finds = 0, g_stat_hops = 0,
                              g_stat_maxhops = 0;
// per K2 task (profiling harness): [0] union walk steps, [1] find hops, [2] link
// retries, [3] rounds (task = blockIdx.x * 8 + warp)
__device__ unsigned* g_k2_taskstat = nullptr;
#define CCL_STAT(v) atomicAdd(&(v), 1ull)
#define CCL_TASKSTAT(k, n) (g_k2_taskstat ? (void)atomicAdd(g_k2_taskstat + 4 * (blockIdx.x * unsigned(CCL_K2_WARPS) + (threadIdx.x >> 5)) + (k), (n)) : (void)0)
#else
#define CCL_STAT(v) ((void)0)
#define CCL_TASKSTAT(k, n) ((void)0)
#endif

// Global min-union (reading R11).  The finds use L1-cacheable loads: many
// unions of a giant component end at the same root, and serving that hot
// entry from each SM's L1 instead of one L2 slice removes the serialisation
// that dominated this kernel.  A stale L1 value is an older parent, i.e. a
// higher ancestor-or-self of the current one: a find may then stop at a node
// that was a root but no longer is -- the atomicMin link detects that
// (returns old != root) and the union continues from the true parent.  Two
// nodes found under one (possibly stale) root are in one set, since sets only
// ever merge.  Path halving stores write ancestors; a halving store can only
// overwrite an atomicMin made on an already non-root node, whose issuer
// re-unions from the value it displaced.  Every root is its set's minimum.
__device__ __forceinline__ int ld_ca(const int32_t* p) {
    int v;
    asm volatile("ld.global.ca.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ void red_min(int32_t* p, int v) {
    asm volatile("red.relaxed.gpu.global.min.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

#ifndef CCL_K2_FULLC
#define CCL_K2_FULLC 0
#endif
__device__ __forceinline__ int find_g(int32_t* G, int a) {
#if CCL_K2_FULLC
    // Walk to the root, then point every node of the walk straight at it with
    // fire-and-forget atomic mins (no reply on the critical path).  A min can
    // never undo a newer link (it only lowers an entry, and every value it
    // writes is an ancestor in the node's set), so stale L1 reads cannot lose
    // a union; chains that concurrent min-links string through the bands are
    // cut for every later walker after the first.
    int x = a, p = ld_ca(G + a);
    CCL_LOOP_GUARD(fgc);
    while (p != x) {
        CCL_LOOP_TICK(fgc);
        x = p;
        p = ld_ca(G + x);
    }
    int y = a;
    CCL_LOOP_GUARD(fgc2);
    while (y > x) {
        CCL_LOOP_TICK(fgc2);
        const int next = ld_ca(G + y);
        red_min(G + y, x);
        y = next;
    }
    return x;
#else
    int p = ld_ca(G + a);
    CCL_LOOP_GUARD(fgh);
#ifdef CCL_STATS
    unsigned long long hops = 0;
    atomicAdd(&g_stat_finds, 1ull);
#endif
    while (p != a) {
        CCL_LOOP_TICK(fgh);
#ifdef CCL_STATS
        ++hops;
#endif
        const int gp = ld_ca(G + p);
        if (gp != p) st_volatile(G + a, gp);
        a = p;
        p = gp;
    }
#ifdef CCL_STATS
    atomicAdd(&g_stat_hops, hops);
    atomicMax(&g_stat_maxhops, hops);
    CCL_TASKSTAT(1, unsigned(hops));
#endif
    return a;
#endif
}
// (A two-pass full path compression here -- rewriting every visited node to
// the root found through possibly stale L1 values -- lost unions under heavy
// contention (percolation noise) and was dropped; halving stores only ever
// write a grandparent read one step earlier.)

__device__ __forceinline__ void union_g(int32_t* G, int a, int b) {
    CCL_STAT(g_stat_unions);
    CCL_LOOP_GUARD(ug);
    while (true) {
        CCL_LOOP_TICK(ug);
        CCL_STAT(g_stat_steps);
        CCL_TASKSTAT(0, 1u);
        a = find_g(G, a);
        b = find_g(G, b);
        if (a == b) return;
        if (a < b) { int t = a; a = b; b = t; }
        const int old = atomicMin(G + a, b);
        if (old == a) return;
        CCL_TASKSTAT(2, 1u);
        a = old;
    }
}

// Read-only find for after all unions are done (L1-cacheable loads: the hot
// root of a giant component is then served from each SM's L1).
__device__ __forceinline__ int find_g_ro(const int32_t* G, int a) {
    int p = __ldg(G + a);
    CCL_LOOP_GUARD(fg);
#ifdef CCL_STATS
    unsigned long long hops = 0;
    atomicAdd(&g_stat_finds, 1ull);
#endif
    while (p != a) {
#ifdef CCL_STATS
        ++hops;
#endif
        CCL_LOOP_TICK(fg);
        CCL_ASSERT(p >= 0 && p < a);
        a = p;
        p = __ldg(G + a);
    }
#ifdef CCL_STATS
    atomicAdd(&g_stat_hops, hops);
    atomicMax(&g_stat_maxhops, hops);
#endif
    return a;
}

// ------------------------------------------------------------- tile decode
struct TileId {
    int b, tx, ty, x0, y0;
};

template <int TY>
__device__ __forceinline__ TileId decode_tile(const Geom& g, unsigned t) {
    TileId id;
    const unsigned q = g.div_tx.div(t);
    id.tx = int(t - q * unsigned(g.tiles_x));
    const unsigned q2 = g.div_ty.div(q);
    id.ty = int(q - q2 * unsigned(g.tiles_y));
    id.b = int(q2);
    id.x0 = id.tx * kTileW;
    id.y0 = id.ty * TY;
    return id;
}

// ---------------------------------------------- edge-slot union-find (K2)
// G[s] = (X << 32) | parent slot, X = the parent's raster index (a root: its
// own).  Same protocol as the 32-bit raster-indexed form it replaces (reading
// R11: lock-free minimum-root union, retry from the displaced parent, path
// halving that only ever stores an ancestor's entry), with the order "smaller
// raster index" carried in the high word so one 64-bit atomicMin links.
__device__ __forceinline__ uint64_t ld_ca64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_volatile64(uint64_t* p, uint64_t v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Root entry of slot a's set (path halving: a re-pointed at its grandparent).
__device__ __forceinline__ uint64_t find_e(uint64_t* G, unsigned a) {
    uint64_t v = ld_ca64(G + a);
    CCL_LOOP_GUARD(fe);
#ifdef CCL_STATS
    unsigned long long hops = 0;
    atomicAdd(&g_stat_finds, 1ull);
#endif
    while (unsigned(v) != a) {
        CCL_LOOP_TICK(fe);
#ifdef CCL_STATS
        ++hops;
#endif
        const unsigned p = unsigned(v);
        const uint64_t w = ld_ca64(G + p);  // p's entry: its parent (the grandparent)
        if (unsigned(w) != p) st_volatile64(G + a, w);
        a = p;
        v = w;
    }
#ifdef CCL_STATS
    atomicAdd(&g_stat_hops, hops);
    atomicMax(&g_stat_maxhops, hops);
    CCL_TASKSTAT(1, unsigned(hops));
#endif
    return v;
}

__device__ __forceinline__ void union_e(uint64_t* G, unsigned a, unsigned b) {
    CCL_STAT(g_stat_unions);
    CCL_LOOP_GUARD(ue);
    while (true) {
        CCL_LOOP_TICK(ue);
        CCL_STAT(g_stat_steps);
        CCL_TASKSTAT(0, 1u);
        uint64_t va = find_e(G, a), vb = find_e(G, b);
        if (va == vb) return;  // one root (distinct roots have distinct raster indices)
        if (va < vb) { const uint64_t t = va; va = vb; vb = t; }
        const uint64_t old = atomicMin(reinterpret_cast<unsigned long long*>(G + unsigned(va)),
                                       static_cast<unsigned long long>(vb));
        if (old == va) return;  // va's root was still a root: linked under vb's
        CCL_TASKSTAT(2, 1u);
        a = unsigned(old);  // it had been re-linked: union what the atomicMin displaced
        b = unsigned(vb);
    }
}

// Read-only find over edge slots after all unions (L2 loads).
__device__ __forceinline__ uint64_t find_e_ro(const uint64_t* G, unsigned a) {
    uint64_t v = __ldcg(reinterpret_cast<const unsigned long long*>(G) + a);
    CCL_LOOP_GUARD(fer);
    while (unsigned(v) != a) {
        CCL_LOOP_TICK(fer);
        a = unsigned(v);
        v = __ldcg(reinterpret_cast<const unsigned long long*>(G) + a);
    }
    return v;
}

// Warp-cooperative union of a batch of root pairs: each lane holds at most one
// pair (a, b) (a < 0: none).  Pairs already seen in this warp are dropped
// (identical root pairs are common: two large components meet at many places
// along a tile edge) so only one lane per distinct pair runs the union.
template <bool NOUNION = false>
__device__ __forceinline__ void warp_union_pairs(uint64_t* G, int a, int b, unsigned long long& last) {
    if (a > b) { int t = a; a = b; b = t; }
    const unsigned long long key =
        (a >= 0 && a != b) ? ((unsigned long long)(unsigned)a << 32) | (unsigned)b : ~0ull;
    const unsigned grp = __match_any_sync(kFull, key);
    const int lane = threadIdx.x & 31;
    if (!NOUNION && key != ~0ull && key != last && (__ffs(grp) - 1) == lane) union_e(G, unsigned(a), unsigned(b));
    if (key != ~0ull) last = key;
}

// edge slot of a K1 run record's root (boundary-row runs always carry a tag)
__device__ __forceinline__ int rec_slot(uint32_t rec, unsigned ntiles, size_t t) {
    CCL_ASSERT((rec >> 16) != 0);
    return int(edge_slot(ntiles, int(rec >> 16) - 1, unsigned(t)));
}

// image-local raster index of a K1 run record's root (tile origin x0, y0)
__device__ __forceinline__ int rec_root(uint32_t rec, int W, int x0, int y0) {
    const int rr = int(rec & 0x7FFFu);
    return (y0 + (rr >> 10)) * W + x0 + (rr & 1023);
}

__device__ __forceinline__ size_t tile_index(const Geom& g, int b, int ty, int tx) {
    return (size_t(b) * g.tiles_y + ty) * g.tiles_x + tx;
}

// =========================================================== K1: local merge
// The tile's foreground is first turned into compact run lists (one entry per
// row run, in raster order of the run starts) so every later step -- local UF,
// flatten, edge output, per-run records -- runs one thread per run with all
// lanes busy, instead of looping over the set bits of each lane's mask word.
//
// Coarse labeling (Alg. 1 l.9-24): the row scan + row-column unification in
// the row direction is exact here -- every pixel's provisional label is its
// run, the lowest equivalent label of its row segment.
// Local UF (Alg. 1 l.25-33): each run of row r >= 1 finds the runs of row r-1
// it touches in O(1) from the masks (they are a contiguous index range of the
// sorted upper run list) and min-unions with each (8-conn widens the contact
// interval by one pixel on both sides: the NW / NE diagonals, reading R2/R10).
// Persistent: each block walks tiles t = blockIdx.x, +gridDim.x, ...; the
// 128-bit image loads of the NEXT tile are issued into registers before the
// current tile is processed, so HBM reads overlap the shared-memory work.

// One 32-px mask word of a K1 tile row.
struct __align__(16) WordE {
    uint32_t m;    // foreground mask
    uint32_t s;    // run-start mask (tile-local runs)
    uint32_t e;    // run-end mask
    int32_t pad;   // number of run starts in the row before this word
};

// Run lists of a tile live in shared memory up to k1_cap runs (natural
// images: a few hundred; i.i.d. noise at density 1/2: ~4096), which keeps the
// block at 45 KB -- with one prefetch register set (44 registers) 5 blocks
// (40 warps) per SM; measured: 4 blocks 46.8 us, 5 blocks 43.6 us on C3
// texture (a cap of 4096 also allowed 5 blocks but sent half the noise tiles
// to the scratch path).  A tile with more runs (period-2 stripes,
// checkerboards: up to TY*512) keeps them in the block's slot of a global
// scratch area instead (same code, L2-resident).
#ifndef CCL_K1_CAP16
#define CCL_K1_CAP16 4576
#endif
#ifndef CCL_K1_SCFENCE
#define CCL_K1_SCFENCE 0  // a fence.sc before the ready flag (measured 0.3 us slower; the release suffices)
#endif
#ifndef CCL_K1_DENSE_FROMBITS
#define CCL_K1_DENSE_FROMBITS 0  // deferred run-dense tiles: masks read back from the bit mask
#endif
#ifndef CCL_K1_STEAL
#define CCL_K1_STEAL 1  // union phase: runs beyond the first T1 in dynamic chunks of 32 per warp
#endif
#ifndef CCL_K1_UF2
#define CCL_K1_UF2 0  // two-step local UF (up-link forest, then the remaining pairs)
#endif
template <int TY>
__host__ __device__ constexpr int k1_min_blocks() {
    return TY > 16 ? (CCL_K1_T32 == 512 ? 2 : CCL_K1_BLOCKS32) : CCL_K1_BLOCKS;
}

template <int TY>
struct K1Smem {
    WordE wd[TY][kWords];
    uint16_t rs[k1_cap<TY>() + 8];  // run k: start x | row << 10; rs[total] = sentinel row 63
    uint16_t re[k1_cap<TY>() + 8];  // run k: end x
    // parent over tile run ids (min-root forest).  After the flatten, a root
    // whose component touches a tile edge carries bit 31 and (1 + its
    // edge-list index) << 16; the low 16 bits are always the parent id.
    int32_t P[k1_cap<TY>()];
    int32_t ecount;                // edge-list length
    int32_t lc[TY], rc[TY];        // roots of the left / right column pixels
    int32_t rcnt[TY];              // runs per row
    int32_t rbase[TY + 1];         // first run id of each row (exclusive prefix)
    int32_t ndefer;                // run-dense tiles of this block (listed in g.defer), labelled last
    int32_t unext;                 // union phase: next unclaimed chunk of 32 runs (CCL_K1_STEAL)
};

// find / merge of §2.1.3 over tile run ids.
#ifdef CCL_STATS
__device__ unsigned long long g_stat_k1_unions = 0, g_stat_k1_steps = 0, g_stat_k1_hops = 0;
#endif
__device__ __forceinline__ int find_r(int32_t* P, int a) {
    volatile int32_t* V = P;
    int p = V[a];
    CCL_LOOP_GUARD(fr);
    while (p != a) {
        CCL_LOOP_TICK(fr);
        CCL_STAT(g_stat_k1_hops);
        const int gp = V[p];
        if (gp != p) V[a] = gp;  // path halving: re-point at an ancestor
        a = p;
        p = gp;
    }
    return a;
}

// read-only find during the flatten: edge tags may be landing on roots, so
// only the low 16 bits (the parent id) are followed
__device__ __forceinline__ int find_r_ro(const int32_t* P, int a) {
    const volatile int32_t* V = P;
    int p = V[a] & 0xFFFF;
    CCL_LOOP_GUARD(fro);
    while (p != a) {
        CCL_LOOP_TICK(fro);
        a = p;
        p = V[a] & 0xFFFF;
    }
    return a;
}

// Lock-free minimum-root union (reading R11): the larger root is re-pointed at
// the smaller with atomicMin; if someone else re-linked it first, retry with
// the value it was linked to.
__device__ __forceinline__ void union_r(int32_t* P, int a, int b) {
    CCL_STAT(g_stat_k1_unions);
    while (true) {
        CCL_STAT(g_stat_k1_steps);
        a = find_r(P, a);
        b = find_r(P, b);
        if (a == b) return;
        if (a < b) { int t = a; a = b; b = t; }
        const int old = atomicMin(&P[a], b);
        if (old == a) return;
        a = old;
    }
}

// K1's union call; profiling variants (DBG bit 8: skipped, bit 16: one
// atomicMin without finds -- timing only, the labels are then wrong).
template <int DBG>
__device__ __forceinline__ void k1_union(int32_t* P, int a, int b) {
    if (DBG & 8) return;
    if (DBG & 16) {
        atomicMin(&P[a], b);
        return;
    }
    union_r(P, a, b);
}

// Profiling builds only (DBG bit 2): per-tile phase timestamps.
__device__ unsigned long long* g_k1_stamps = nullptr;
__device__ unsigned long long* g_k3_stamps = nullptr;
__device__ unsigned long long* g_k2_stamps = nullptr;  // per K2 task: start, end (globaltimer ns)
__device__ unsigned long long* g_k2_phase = nullptr;   // per horizontal K2 task: masks in, records in, 1st batch done
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Timeline of one fused step (profiling builds only, -DCCL_TIMELINE; read by
// ccl_debug_timeline): globaltimer ns of 0 K1 first block start, 1 K1 last
// block end, 2 K2 first task start, 3 K2 last task end, 4 K3 first block
// start, 5 K3 first block past its PDL wait, 6 K3 last block end, 7 K1 last
// tile published.
#ifdef CCL_TIMELINE
__device__ unsigned long long g_tl[8];
__device__ unsigned long long* g_tile_pub = nullptr;  // per tile: globaltimer at its publish
#define CCL_TL_MIN(i) atomicMin(&g_tl[i], gtimer())
#define CCL_TL_MAX(i) atomicMax(&g_tl[i], gtimer())
#else
#define CCL_TL_MIN(i) ((void)0)
#define CCL_TL_MAX(i) ((void)0)
#endif
__device__ __forceinline__ void k1_stamp(unsigned t, int k) {
    if (g_k1_stamps) g_k1_stamps[size_t(t) * 8 + k] = clock64();
}
__device__ __forceinline__ void k3_stamp(unsigned t, int k) {
    if (g_k3_stamps) g_k3_stamps[size_t(t) * 8 + k] = clock64();
}

// rows per warp, and how many of them are prefetched into registers one tile
// ahead: all of them for 8- and 16-row tiles; none for 32-row tiles, whose
// four rows per warp are loaded at the start of their tile from L2 (the next
// tile is pulled into L2 with bulk prefetches one tile ahead) -- measured on
// C3 texture, 5 blocks/SM: 102.4 us/step vs 104.7 with two rows held in
// registers and two loaded in place (CCL_K1_PF32=2), 105.4 with that at 4
// blocks/SM (64 registers)
template <int TY>
__host__ __device__ constexpr int k1_rows_per_warp() { return (TY + k1_warps<TY>() - 1) / k1_warps<TY>(); }
#ifndef CCL_K1_PF32
#define CCL_K1_PF32 0
#endif
template <int TY>
__host__ __device__ constexpr int k1_pf_rows() {
    return k1_rows_per_warp<TY>() <= 2 ? k1_rows_per_warp<TY>() : CCL_K1_PF32;
}

template <int TY>
struct ImgRegs {
    uint4 v[k1_pf_rows<TY>() > 0 ? k1_pf_rows<TY>() : 1][2];  // row i of the warp: bytes 32*lane .. 32*lane + 31
};


// One lane's 32 contiguous pixels of a tile row: one 256-bit load when the
// row is 32-byte aligned (W % 32 == 0 and an aligned image), else two 128-bit
// loads (the row is 16-byte aligned on the vector path); pixels at or beyond
// W read as background.  A warp instruction covers the whole 1024-px row.
__device__ __forceinline__ void ld_px32(const uint8_t* p, int avail, bool v8, uint4& a, uint4& b) {
    a = b = make_uint4(0, 0, 0, 0);
    if (avail >= 32 && v8) {
        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                     : "l"(p));
    } else {
        if (avail >= 16) a = ld_stream_u4(p);
        if (avail >= 32) b = ld_stream_u4(p + 16);
    }
}

template <int TY>
__device__ __forceinline__ void k1_prefetch(const uint8_t* img, const Geom& g, unsigned t, int warp,
                                            int lane, bool v8, ImgRegs<TY>& pf) {
    const TileId id = decode_tile<TY>(g, t);
    const uint8_t* im = img + size_t(id.b) * size_t(g.npx);
#pragma unroll
    for (int i = 0; i < k1_pf_rows<TY>(); ++i) {
        const int y = (warp + i * k1_warps<TY>() < TY) ? id.y0 + warp + i * k1_warps<TY>() : g.H;
        pf.v[i][0] = pf.v[i][1] = make_uint4(0, 0, 0, 0);
        const int x = id.x0 + 32 * lane;
        if (y < g.H) ld_px32(im + size_t(y) * size_t(g.W) + x, g.W - x, v8, pf.v[i][0], pf.v[i][1]);
    }
}

// Row r's mask word for this lane -> start / end masks, row-local run offsets.
template <int TY>
__device__ __forceinline__ void k1_row_init(K1Smem<TY>& sm, int r, int lane, uint32_t m) {
    uint32_t pm = __shfl_up_sync(kFull, m, 1), nm = __shfl_down_sync(kFull, m, 1);
    if (lane == 0) pm = 0;
    if (lane == 31) nm = 0;
    const uint32_t s = m & ~((m << 1) | (pm >> 31));
    const uint32_t e = m & ~((m >> 1) | (nm << 31));
    const int n = __popc(s);
    int incl = n;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += t;
    }
    sm.wd[r][lane] = WordE{m, s, e, incl - n};
    if (lane == 31) sm.rcnt[r] = incl;
}

// K1 from the run lists on: rs / re / P are the block's shared arrays or, for
// a tile over k1_cap runs, its global scratch slot.
// K1 on the rows [r0, r1) of a tile whose runs fit the shared-memory lists
// (every tile is one such range unless it has more than k1_cap runs, e.g.
// i.i.d. noise in 32-row tiles or period-2 stripes: then maximal row ranges
// that fit, one after another).  Run ids are range-local (tile run id - base);
// the records land at their tile run ids.  A range boundary inside the tile
// is treated like a tile edge (its rows' roots become edge slots) and its
// crossing edges are unioned in G by k1_internal_boundary.  ebase = the first
// edge index of this range (a multiple of 4: whole 32-byte slot sectors).
template <int TY, int CONN, int DBG, bool WHOLE>
__device__ __forceinline__ int k1_range(K1Smem<TY>& sm, const Geom& g, unsigned t, const TileId& id, int v,
                                         int r0_, int r1_, int ebase_, uint64_t* G, uint32_t* R, int32_t* E,
                                         int32_t* F, int warp, int lane) {
    constexpr int T1 = k1_threads<TY>(), NW1 = k1_warps<TY>();
    // WHOLE: the tile is one range (every tile of a natural image): constant
    // bounds, so the address arithmetic folds as before the ranges existed
    const int r0 = WHOLE ? 0 : r0_, r1 = WHOLE ? TY : r1_, ebase = WHOLE ? 0 : ebase_;
    uint16_t* __restrict__ rs = sm.rs;
    uint16_t* __restrict__ re = sm.re;
    int32_t* P = sm.P;
    const int tid = threadIdx.x;
    const int b0 = __shfl_sync(kFull, v, max(r0 - 1, 0));
    const int base = r0 > 0 ? b0 : 0;                        // tile run id of the range's first run
    const int total = __shfl_sync(kFull, v, r1 - 1) - base;  // runs of the range
    // run lists: rs / re in raster order of the starts, P[k] = k
#pragma unroll
    for (int i = 0; i < (TY + NW1 - 1) / NW1; ++i) {
        const int r = r0 + warp + i * NW1;
        if (r >= r1) break;  // warp-uniform
        const int rbr = __shfl_sync(kFull, v, max(r - 1, 0));
        const int rb = (r > 0 ? rbr : 0) - base;
        const WordE w = sm.wd[r][lane];
        sm.wd[r][lane].pad = rb + w.pad;  // from here on: range run id of the word's first start
        const int xb = lane << 5;
        int ks = rb + w.pad;
        int ke = ks - ((w.m & 1u) && !(w.s & 1u));  // a run open at the word start ends here
        uint32_t sb = w.s, eb = w.e;
        while (sb) {
            const int bit = __ffs(sb) - 1;
            sb &= sb - 1;
            rs[ks] = uint16_t((xb + bit) | (r << 10));
#if !CCL_K1_UF2
            P[ks] = ks;
#endif
            ++ks;
        }
        while (eb) {
            const int bit = __ffs(eb) - 1;
            eb &= eb - 1;
            re[ke++] = uint16_t(xb + bit);
        }
    }
    if (tid == 0) {
        rs[total] = uint16_t(63 << 10);  // no run of any row: ends every neighbour search
        sm.unext = T1;  // dynamic union chunks start after the static first pass
    }
    __syncthreads();
    if ((DBG & 4) && threadIdx.x == 0) k1_stamp(t, 2);
    if (DBG & 1) {
        __syncthreads();
        return ebase;
    }

    // local UF.  The adjacencies between two rows form a monotone staircase of
    // run pairs; every pair is (k, first upper neighbour of k) or (first lower
    // neighbour of j, j) -- if j is the 2nd+ upper neighbour of k, j starts
    // right of k's start, so it cannot reach k-1.  Each run therefore does at
    // most two unions, found in O(1) from the masks: no fan-in serialisation.
    constexpr int D = CONN == 8 ? 1 : 0;
#if CCL_K1_UF2
    // Column-direction coarse labeling first (Alg. 1 l.14-24 at run level,
    // the A/B of profiles/r02_coarse_labeling_ab.txt): U1 links every run to
    // its first upper neighbour with a plain store (a forest whose roots are
    // their trees' minima), U2 unions only the remaining adjacencies.
#pragma unroll 1
    for (int k = tid; k < total; k += T1) {
        const int rsk = rs[k];
        const int r = rsk >> 10, si = rsk & 1023, ei = re[k];
        const int p = max(si - D, 0), q = min(ei + D, kTileW - 1);
        int parent = k;
        if (r > r0) {
            const WordE uu = sm.wd[r - 1][p >> 5];
            const uint32_t below = (1u << (p & 31)) - 1u;
            const int ju = uu.pad - ((uu.m & 1u) && !(uu.s & 1u)) + __popc(uu.e & below);
            const int rsu = rs[ju];
            if ((rsu >> 10) == r - 1 && (rsu & 1023) <= q) parent = ju;
        }
        P[k] = parent;
    }
    __syncthreads();
#pragma unroll 1
    for (int k = tid; k < total; k += T1) {
        const int rsk = rs[k];
        const int r = rsk >> 10, si = rsk & 1023, ei = re[k];
        if (r + 1 >= r1 || k == 0) continue;
        const int p = max(si - D, 0), q = min(ei + D, kTileW - 1);
        const WordE ud = sm.wd[r + 1][p >> 5];
        const uint32_t below = (1u << (p & 31)) - 1u;
        const int jd = ud.pad - ((ud.m & 1u) && !(ud.s & 1u)) + __popc(ud.e & below);
        const int rsd = rs[jd], rsp = rs[k - 1], ep = re[k - 1];
        // jd touches k, and run k-1 (same row) touches jd too: k is a 2nd+ upper neighbour of jd
        if ((rsd >> 10) == r + 1 && (rsd & 1023) <= q && (rsp >> 10) == r && ep + D >= (rsd & 1023))
            k1_union<DBG>(P, jd, k);
    }
#else
    // run k's two unions: the first runs of rows r-1 and r+1 touching its
    // contact interval [p, q] (both searches are issued before either union:
    // the phase is bound by this chain)
    auto run_unions = [&](int k) {
        const int rsk = rs[k];
        const int r = rsk >> 10, si = rsk & 1023, ei = re[k];
        const int p = max(si - D, 0), q = min(ei + D, kTileW - 1);
        const WordE uu = sm.wd[r > r0 ? r - 1 : r0][p >> 5];
        const WordE ud = sm.wd[r + 1 < r1 ? r + 1 : r1 - 1][p >> 5];
        const uint32_t below = (1u << (p & 31)) - 1u;
        const int ju = uu.pad - ((uu.m & 1u) && !(uu.s & 1u)) + __popc(uu.e & below);
        const int jd = ud.pad - ((ud.m & 1u) && !(ud.s & 1u)) + __popc(ud.e & below);
        const int rsu = rs[ju], rsd = rs[jd];  // may be another row's run or the sentinel
        if (r > r0 && (rsu >> 10) == r - 1 && (rsu & 1023) <= q) k1_union<DBG>(P, k, ju);
        if (r + 1 < r1 && (rsd >> 10) == r + 1 && (rsd & 1023) <= q) k1_union<DBG>(P, jd, k);
    };
#if CCL_K1_STEAL
    // the first T1 runs one per thread; beyond them (run-dense tiles) chunks
    // of 32 runs from a shared counter, so warps whose unions finish early
    // take more -- the phase ends at a barrier, i.e. at its slowest warp (on
    // i.i.d. noise 44 % of K1's stall samples were barrier waits)
    if (tid < total) run_unions(tid);
    if (total > T1) {  // block-uniform
#pragma unroll 1
        for (;;) {
            int k0 = 0;
            if (lane == 0) k0 = atomicAdd(&sm.unext, 32);
            k0 = __shfl_sync(kFull, k0, 0);
            if (k0 >= total) break;
            if (k0 + lane < total) run_unions(k0 + lane);
        }
    }
#else
#pragma unroll 1
    for (int k = tid; k < total; k += T1) run_unions(k);
#endif
#endif
    __syncthreads();
    if ((DBG & 4) && threadIdx.x == 0) k1_stamp(t, 3);
    // flatten + Alg. 1 l.34-39 for tile-edge items only (reading R7 for the
    // index conversion): every run points at its root; the first run to find
    // that its root's component touches a tile edge (top / bottom row run,
    // left / right column pixel, or a row next to a range boundary) claims the
    // root (bit 31), takes the next edge index i of the tile and tags the root
    // with 1 + i (claim order: any bijection works, the labels do not depend
    // on it); the root becomes edge slot i * ntiles + t with entry (global
    // raster index << 32) | slot.
    if ((DBG & 4) && threadIdx.x == 0) k1_stamp(t, 4);
    const int W = g.W, x0 = id.x0, y0 = id.y0;
    const int last_row = min(TY, g.H - y0) - 1;  // (r1 - 1 >= last_row for the last range)
    const int rl = min(r1 - 1, last_row);
    // rows that border another tile (or, in strip mode, another strip) or range
    const bool top = r0 > 0 || y0 > 0 || g.force_top;
    const bool bottom = rl < last_row || y0 + TY < g.H || (g.force_bottom && y0 + TY >= g.H);
    const bool left = x0 > 0, right = x0 + kTileW < W;
    int32_t* Eh = E + size_t(t) * kEdgeCap;
#pragma unroll 1
    for (int k = tid; k < total; k += T1) {  // (chunked work stealing here measured slower: 101.6 vs 100.7 us)
        const int root = find_r_ro(P, k);
        if (root != k) P[k] = root;  // an ancestor: concurrent finds stay valid
        const int rsk = rs[k];
        const int r = rsk >> 10, si = rsk & 1023, ei = re[k];
        const bool hrow = (r == r0 && top) || (r == rl && bottom);
        const bool lc = si == 0 && left, rc = ei == kTileW - 1 && right;
        if (hrow || lc || rc) {
            if (!(atomicOr(&P[root], int(0x80000000u)) & int(0x80000000u))) {
                const int idx = ebase + atomicAdd(&sm.ecount, 1);
                CCL_ASSERT(idx < edge_slots(TY));
                P[root] = root | int(0x80000000u) | ((idx + 1) << 16);
            }
            if (lc) sm.lc[r] = k;  // the column pixel's run (its root's slot after the claims)
            if (rc) sm.rc[r] = k;
        }
    }
    if (DBG & 2) {
        __syncthreads();
        __syncthreads();
        return ebase;
    }
    __syncthreads();
    if ((DBG & 4) && threadIdx.x == 0) k1_stamp(t, 5);
    // edge brief: header, column-root slots of the range's rows; per-run
    // records for K3 / K2
    const int ne = ebase + sm.ecount;  // (read before the last barrier: the next range / tile resets it)
    const int rbl = __shfl_sync(kFull, v, max(last_row - 1, 0));
    const int rb_last = last_row > 0 ? rbl : 0;  // tile run id of the last valid row's first run
    if (tid == 0) {
        st_keep(Eh, ne);
        st_keep(Eh + 1, rb_last);
    }
    for (int j = tid; j < 2 * (r1 - r0); j += T1) {
        const int r = r0 + (j >> 1);
        const int k = (j & 1) ? sm.rc[r] : sm.lc[r];
        int slot = -1;
        if (k >= 0) slot = int(edge_slot(g.ntiles, ((P[P[k] & 0xFFFF] >> 16) & 0x7FFF) - 1, t));
        st_keep(Eh + ((j & 1) ? kEdgeRC : kEdgeLC) + r, slot);
    }
    uint32_t* Rt = R + size_t(t) * runs_per_tile_cap<TY>();
#pragma unroll 1
    for (int k = tid; k < total; k += T1) {
        const int root = P[k] & 0xFFFF;
        const int tag = (P[root] >> 16) & 0x7FFF;  // 1 + edge index, or 0
        const uint32_t rec = uint32_t(rs[root]) | (uint32_t(tag) << 16);
        const int kt = base + k;  // tile run id
        st_keep(Rt + kt, rec);
        // the first kRL runs of the first and last rows again in the edge
        // brief: the boundary analysis' first round trip
        if (kt < kRL) st_keep(reinterpret_cast<uint32_t*>(Eh) + kEdgeR0 + kt, rec);
        if (kt >= rb_last && kt < rb_last + kRL) st_keep(reinterpret_cast<uint32_t*>(Eh) + kEdgeRL + (kt - rb_last), rec);
        // edge index -> root run (re, the run ends, is free after the flatten)
        if (root == k && tag) re[tag - 1 - ebase] = uint16_t(k);
    }
    __syncthreads();  // the slot writes below read rs / re: the next range / tile rewrites them only
                      // after its own first barrier
    if ((DBG & 4) && threadIdx.x == 0) k1_stamp(t, 6);
    // the edge slots' initial entries (raster index << 32 | slot: every edge
    // root its own set), four per thread = one whole 32-byte sector, so the
    // boundary analysis' loads and atomics hit fully valid L2 sectors; a
    // sector's unused tail (edge indices >= ne) holds harmless self-roots
#pragma unroll 1
    for (int j = tid; 4 * j < ne - ebase; j += T1) {
        uint32_t vv[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = ebase + 4 * j + q;
            uint32_t gr = 0x7FFFFFFEu;
            if (i < ne) {
                const int rr = rs[re[i - ebase]];
                gr = uint32_t((y0 + (rr >> 10)) * W + x0 + (rr & 1023));
            }
            // strip marks (ccl_strip.cuh), the padding too: a run-dense tile's
            // next range starts at the next sector, so padding slots lie below
            // the tile's edge count and K3 resolves them (labels never used)
            if (g.strip) F[edge_slot(g.ntiles, i, t)] = -1;
            vv[2 * q] = edge_slot(g.ntiles, i, t);
            vv[2 * q + 1] = gr;
        }
        int4* sec = reinterpret_cast<int4*>(G + edge_slot(g.ntiles, ebase + 4 * j, t));
        st_keep_v4(sec, make_int4(int(vv[0]), int(vv[1]), int(vv[2]), int(vv[3])));
        st_keep_v4(sec + 1, make_int4(int(vv[4]), int(vv[5]), int(vv[6]), int(vv[7])));
    }
    return ne;
}

// Unions of the foreground edges that cross the boundary above row rb of
// tile t (a boundary between two row ranges of one tile): one warp, the
// same pair extraction as the boundary analysis' horizontal tasks, from the
// tile's masks (shared memory) and its just-written run records.
template <int TY, int CONN>
__device__ __forceinline__ void k1_internal_boundary(K1Smem<TY>& sm, const Geom& g, unsigned t, int v, int rb,
                                                     uint64_t* G, const uint32_t* R, int lane) {
    const uint32_t cur = sm.wd[rb][lane].m, up = sm.wd[rb - 1][lane].m;
    uint32_t curL = __shfl_up_sync(kFull, cur, 1), upL = __shfl_up_sync(kFull, up, 1);
    uint32_t curR = __shfl_down_sync(kFull, cur, 1), upR = __shfl_down_sync(kFull, up, 1);
    if (lane == 0) { curL = 0; upL = 0; }
    if (lane == 31) { curR = 0; upR = 0; }
    const uint32_t sc = cur & ~((cur << 1) | (curL >> 31)), su = up & ~((up << 1) | (upL >> 31));
    int ic = __popc(sc), iu = __popc(su);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int a = __shfl_up_sync(kFull, ic, d), c = __shfl_up_sync(kFull, iu, d);
        if (lane >= d) { ic += a; iu += c; }
    }
    ic -= __popc(sc);
    iu -= __popc(su);
    const uint32_t o = cur & up, oL = curL & upL;
    uint32_t ev = o & ~((o << 1) | (oL >> 31));
    uint32_t ne = 0, nw = 0;
    if (CONN == 8) {
        const uint32_t cur_n = (cur >> 1) | (curR << 31), up_n = (up >> 1) | (upR << 31);
        const uint32_t cur_p = (cur << 1) | (curL >> 31), up_p = (up << 1) | (upL >> 31);
        ne = cur & ~cur_n & ~up & up_n;
        nw = cur & ~cur_p & ~up & up_p;
    }
    const uint32_t* Rt = R + size_t(t) * runs_per_tile_cap<TY>();
    const int base_c = __shfl_sync(kFull, v, rb - 1);  // tile run id of row rb's first run
    const int bu = __shfl_sync(kFull, v, max(rb - 2, 0));
    const int base_u = rb > 1 ? bu : 0;                  // ... of row rb - 1
    unsigned long long last = ~0ull;
    // the run containing pixel x of a row (word data of that row from a shuffle)
    auto run_of = [&](uint32_t s, int pad, int x) {
        const uint32_t sw = __shfl_sync(kFull, s, x >> 5);
        const int pw = __shfl_sync(kFull, pad, x >> 5);
        return pw + __popc(sw & (kFull >> (31 - (x & 31)))) - 1;
    };
    while (__any_sync(kFull, ev | ne | nw)) {
        int x = 0, xu = 0;
        const bool have = (ev | ne | nw) != 0;
        if (ev) {
            x = (lane << 5) + __ffs(ev) - 1;
            ev &= ev - 1;
            xu = x;
        } else if (ne) {
            x = (lane << 5) + __ffs(ne) - 1;
            ne &= ne - 1;
            xu = x + 1;
        } else if (nw) {
            x = (lane << 5) + __ffs(nw) - 1;
            nw &= nw - 1;
            xu = x - 1;
        }
        // every lane takes part in the shuffles (x = 0 for lanes without an event)
        const int ia = run_of(sc, ic, x), ib = run_of(su, iu, xu);
        int a = -1, b = -1;
        if (have) {
            a = rec_slot(__ldcg(Rt + base_c + ia), g.ntiles, t);
            b = rec_slot(__ldcg(Rt + base_u + ib), g.ntiles, t);
        }
        warp_union_pairs(G, a, b, last);
    }
}


// K1, first half of a tile: pixels -> masks, row runs, run numbering.
// Returns v (lane r: tile run id of the first run of row r + 1).  INPLACE:
// the tile's pixels are loaded here (run-dense tiles, processed after the
// block's other tiles); else they were prefetched into cur, which then
// receives the next tile.
template <int TY, int CONN, bool VEC, bool INPLACE, int DBG = 0, int THR = 0>
__device__ __forceinline__ int k1_masks(K1Smem<TY>& sm, const uint8_t* img, const Geom& g, unsigned t,
                                        ImgRegs<TY>& cur, unsigned tnext, unsigned ntiles, uint32_t* bits,
                                        int warp, int lane, bool v8) {
    const TileId id = decode_tile<TY>(g, t);
    const uint8_t* im = img + size_t(id.b) * size_t(g.npx);
    uint32_t* bm = bits + size_t(id.b) * size_t(g.nwords);
    const int tid = threadIdx.x;
    if ((DBG & 4) && threadIdx.x == 0) k1_stamp(t, 0);

    // Alg. 1 l.3-8: the tile's pixels -> foreground masks (out-of-image pixels
    // read as background, R5).  The rows not held in the prefetch registers
    // (32-row tiles: the warp's last two; INPLACE: all) are loaded first.
    constexpr int RPW = k1_rows_per_warp<TY>(), PFR = INPLACE ? 0 : k1_pf_rows<TY>();
    constexpr int NL = RPW - PFR > 0 ? RPW - PFR : 1;
    // INPLACE (a deferred run-dense tile): its masks were written by the main
    // loop's pass over it -- read them back from L2 instead of the image
    constexpr bool FROMBITS = INPLACE && CCL_K1_DENSE_FROMBITS;
    uint4 lv[NL][2];
    if (VEC && !FROMBITS) {
#pragma unroll
        for (int i = PFR; i < RPW; ++i) {
            const int r = warp + i * k1_warps<TY>(), y = id.y0 + r, x = id.x0 + 32 * lane;
            lv[i - PFR][0] = lv[i - PFR][1] = make_uint4(0, 0, 0, 0);
            if (r < TY && y < g.H) ld_px32(im + size_t(y) * size_t(g.W) + x, g.W - x, v8, lv[i - PFR][0], lv[i - PFR][1]);
        }
    }
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int r = warp + i * k1_warps<TY>();
        if (r >= TY) break;  // warp-uniform
        const int y = id.y0 + r;
        uint32_t m = 0;
        const int wg = id.tx * kWords + lane;
        if (FROMBITS) {
            m = (y < g.H && wg < g.WW) ? __ldcg(bm + size_t(y) * g.WW + wg) : 0u;
        } else if (VEC) {
            // the lane's own 32 contiguous pixels: no cross-lane assembly
            const uint4 v0 = i < PFR ? cur.v[i < PFR ? i : 0][0] : lv[i >= PFR ? i - PFR : 0][0];
            const uint4 v1 = i < PFR ? cur.v[i < PFR ? i : 0][1] : lv[i >= PFR ? i - PFR : 0][1];
            m = nzc16<THR>(v0, g.thr_k) | (nzc16<THR>(v1, g.thr_k) << 16);
        } else {
            const uint8_t* row = im + size_t(y < g.H ? y : 0) * size_t(g.W);
#pragma unroll 4
            for (int k = 0; k < kWords; ++k) {
                const int x = id.x0 + (k << 5) + lane;
                const bool fg = (y < g.H && x < g.W) ? (THR ? int(row[x]) >= g.thr : row[x] != 0) : false;
                const uint32_t bal = __ballot_sync(kFull, fg);
                if (lane == k) m = bal;
            }
        }
        if (!FROMBITS && y < g.H && wg < g.WW) st_keep(bm + size_t(y) * g.WW + wg, m);
        k1_row_init<TY>(sm, r, lane, m);
    }
    // the pixels are in the masks now: the prefetch registers receive the
    // block's next tile, in flight during the rest of this one ...
    if (!INPLACE && VEC && tnext < ntiles) k1_prefetch<TY>(img, g, tnext, warp, lane, v8, cur);
    // ... and its other rows are pulled into L2 with bulk prefetches
    constexpr int L2R = k1_pf_rows<TY>() * k1_warps<TY>();  // first row pulled into L2
    if (!INPLACE && VEC && RPW > k1_pf_rows<TY>() && tnext < ntiles && warp == k1_warps<TY>() - 1 &&
        lane < TY - L2R) {
        const TileId nx = decode_tile<TY>(g, tnext);
        const int y = nx.y0 + L2R + lane;
        if (y < g.H) {
            const uint8_t* row = img + size_t(nx.b) * size_t(g.npx) + size_t(y) * size_t(g.W) + nx.x0;
            const unsigned bytes = unsigned(min(kTileW, g.W - nx.x0));
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row), "r"(bytes) : "memory");
        }
    }
    if (tid < TY) sm.lc[tid] = -1;
    else if (tid < 2 * TY) sm.rc[tid - TY] = -1;
    else if (tid == 2 * TY) sm.ecount = 0;
    __syncthreads();
    if ((DBG & 4) && threadIdx.x == 0) k1_stamp(t, 1);

    // run numbering: v (lane r) = first run id of row r+1
    int v = lane < TY ? sm.rcnt[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(kFull, v, d);
        if (lane >= d) v += u;
    }
    if (warp == 0 && lane < TY) sm.rbase[lane + 1] = v;
    if (warp == 0 && lane == 0) sm.rbase[0] = 0;
    return v;
}

// K1 publishes a finished tile to the boundary analysis (K1 -> K2 overlap)
__device__ __forceinline__ void k1_publish(const Geom& g, unsigned t) {
    if (g.epoch) {  // every output of the tile is written
        __syncthreads();
        if (threadIdx.x == 0) {
            // the barrier orders the block's writes before this thread's
            // release, which is cumulative at gpu scope (st.release = a
            // fence.acq_rel + the store); CCL_K1_SCFENCE adds a full fence.sc
#if CCL_K1_SCFENCE
            __threadfence();
#endif
            st_release_u64(g.ready + t, g.epoch);
            CCL_TL_MAX(7);
#ifdef CCL_TIMELINE
            if (g_tile_pub) g_tile_pub[t] = gtimer();
#endif
        }
    }
}

// K1, second half of a run-dense tile (more runs than the shared-memory
// lists hold): maximal row ranges that fit, each labelled alone, then the
// range boundaries unioned in G like tile boundaries.
template <int TY, int CONN, int DBG = 0>
__device__ __forceinline__ void k1_dense(K1Smem<TY>& sm, const Geom& g, unsigned t, int v, uint64_t* G, uint32_t* R,
                                         int32_t* E, int32_t* F, int warp, int lane) {
    const int tid = threadIdx.x;
    const TileId id = decode_tile<TY>(g, t);
    // maximal row ranges whose runs fit the shared-memory lists (one range
    // unless the tile is run-dense); each is labelled alone, then the range
    // boundaries are unioned in G like tile boundaries
    int r0 = 0, ebase = 0;
    uint32_t inner = 0;  // rows that start a range after the first
    while (r0 < TY) {  // block-uniform
        const int b0 = __shfl_sync(kFull, v, max(r0 - 1, 0));
        const int base = r0 > 0 ? b0 : 0;
        const unsigned fit = __ballot_sync(kFull, lane >= r0 && lane < TY && v - base <= k1_cap<TY>());
        const int r1 = 32 - __clz(fit);  // >= r0 + 1: one row has <= 512 runs
        if (r0 > 0) {
            inner |= 1u << r0;
            __syncthreads();  // the previous range's slot writes have read rs / re / ecount
            if (tid == 0) sm.ecount = 0;
        }
        const int ne = k1_range<TY, CONN, DBG, false>(sm, g, t, id, v, r0, r1, ebase, G, R, E, F, warp, lane);
        ebase = (ne + 3) & ~3;  // the next range starts on a whole slot sector
        r0 = r1;
    }
    if (inner) {
        __syncthreads();  // every range's records and slot entries are written
        int i = 0;
        for (uint32_t m = inner; m; m &= m - 1, ++i)
            if (warp == i % k1_warps<TY>()) k1_internal_boundary<TY, CONN>(sm, g, t, v, __ffs(m) - 1, G, R, lane);
        __syncthreads();  // (the next tile rewrites the row words these read)
    }
    k1_publish(g, t);
}

// ============================================================ K2: boundary
// Boundary analysis (Alg. 2, §2.2): min-union of the local roots on the two
// sides of every foreground edge that crosses a tile boundary (reading R9 /
// R10).  The local roots come from K1's compact outputs -- the per-run records
// of the tile rows next to a horizontal boundary and the column-root lists of
// the tiles next to a vertical boundary -- so the only scattered accesses are
// the union walks over the roots' parent entries in G.
// K1's outputs are read with ld.global.cg (L2).


// The horizontal boundary above tile (b, band >= 1, tx); one warp.
#ifndef CCL_PAIRS_PER_LANE
#define CCL_PAIRS_PER_LANE 4
#endif
constexpr int kPairsPerLane = CCL_PAIRS_PER_LANE;  // boundary pairs a lane contributes per round

template <int TY, int CONN, bool NOUNION = false>
__device__ __forceinline__ void boundary_h(const Geom& g, const uint32_t* bits, const uint32_t* R,
                                           const int32_t* E, uint64_t* G, int b, int band, int tx,
                                           Word (*s_w)[kWords], int2* pairs, int sub = 0, int sub_log2 = 0) {
    const int lane = threadIdx.x & 31;
    constexpr int RCAP = runs_per_tile_cap<TY>();
    const int x0 = tx * kTileW, y0 = band * TY;
    const size_t t_lo = tile_index(g, b, band, tx);  // tile below the edge
    const size_t t_up = t_lo - g.tiles_x;             // tile above
    const uint32_t* bm = bits + size_t(b) * size_t(g.nwords);
    const uint32_t* Rlo = R + t_lo * RCAP;  // row 0 runs start at run id 0
    const int32_t* Elo = E + t_lo * kEdgeCap;
    const int32_t* Eup = E + t_up * kEdgeCap;
    const bool has_l = tx > 0, has_r = x0 + kTileW < g.W;
    // ---- one round trip for the task's inputs: the two facing mask rows, the
    // first 32 run records of each facing row (from the edge briefs), the
    // corner words and column-root slots, the upper tile's last-row run base
    // (only needed beyond 32 runs in a row)
    const int up_base = __ldcg(Eup + 1);
    const int wg = tx * kWords + lane;
    const uint32_t* rowc = bm + size_t(y0) * g.WW;
    const uint32_t* rowu = rowc - g.WW;
    const uint32_t cur = wg < g.WW ? __ldcg(rowc + wg) : 0u;
    const uint32_t up = wg < g.WW ? __ldcg(rowu + wg) : 0u;
    const uint32_t r0 = uint32_t(__ldcg(Elo + kEdgeR0 + lane));  // records of the lower tile's top-row runs 0..31
    const uint32_t rl = uint32_t(__ldcg(Eup + kEdgeRL + lane));  // ... of the upper tile's last-row runs 0..31
    uint32_t corner = 0;
    int ca = -1, cb = -1;  // tile-corner diagonal pair: slots straight from the column-root lists
    if (CONN == 8 && lane == 0 && has_l) {
        corner = __ldcg(rowu + wg - 1);
        ca = __ldcg(Elo + kEdgeLC);
        cb = __ldcg(Eup - kEdgeCap + kEdgeRC + TY - 1);
    }
    if (CONN == 8 && lane == 31 && has_r) {
        corner = __ldcg(rowu + wg + 1);
        ca = __ldcg(Elo + kEdgeRC);
        cb = __ldcg(Eup + kEdgeCap + kEdgeLC + TY - 1);
    }
    uint32_t curL = __shfl_up_sync(kFull, cur, 1), upL = __shfl_up_sync(kFull, up, 1);
    uint32_t curR = __shfl_down_sync(kFull, cur, 1), upR = __shfl_down_sync(kFull, up, 1);
    if (lane == 0) { curL = 0; upL = 0; }
    if (lane == 31) { curR = 0; upR = 0; }
    const uint32_t sc = cur & ~((cur << 1) | (curL >> 31)), su = up & ~((up << 1) | (upL >> 31));
    // row-local run index of the first start in each word (prefix of popc)
    int ic = __popc(sc), iu = __popc(su);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int a = __shfl_up_sync(kFull, ic, d), c = __shfl_up_sync(kFull, iu, d);
        if (lane >= d) { ic += a; iu += c; }
    }
    s_w[0][lane] = Word{cur, sc, 0, ic - __popc(sc)};
    s_w[1][lane] = Word{up, su, 0, iu - __popc(su)};
    __syncwarp();
#ifdef CCL_K2_PHASES  // profiling harness only (tools/k1_phases.cu)
    const unsigned ptask = blockIdx.x * unsigned(CCL_K2_WARPS) + (threadIdx.x >> 5);
    if (g_k2_phase && lane == 0) g_k2_phase[4 * size_t(ptask)] = gtimer();
#endif
    const uint32_t o = cur & up, oL = curL & upL;
    uint32_t ev = o & ~((o << 1) | (oL >> 31));
    uint32_t ne = 0, nw = 0;
    bool corner_pair = false;
    if (CONN == 8) {
        const uint32_t cur_n = (cur >> 1) | (curR << 31), up_n = (up >> 1) | (upR << 31);
        const uint32_t cur_p = (cur << 1) | (curL >> 31), up_p = (up << 1) | (upL >> 31);
        ne = cur & ~cur_n & ~up & up_n;
        nw = cur & ~cur_p & ~up & up_p;
        if (lane == 0 && has_l && (cur & 1u)) corner_pair = (corner >> 31) != 0;   // (x0, y0) -- (x0-1, y0-1)
        if (lane == 31 && has_r && (cur >> 31)) corner_pair = (corner & 1u) != 0;  // (x0+1023, y0) -- (x0+1024, y0-1)
    }
    if ((lane >> (5 - sub_log2)) != sub) {  // another warp's share of this boundary
        ev = ne = nw = 0;
        corner_pair = false;
    }
    // run index (within its row) of the run containing foreground pixel x:
    // (number of run starts at positions <= x) - 1
    auto run_idx = [&](int row, int x) {
        CCL_ASSERT(x >= 0 && x < kTileW);
        const Word& w = s_w[row][x >> 5];
        const int i = w.pad + __popc(w.s & (kFull >> (31 - (x & 31)))) - 1;
        CCL_ASSERT(i >= 0 && i < kTileW / 2);
        return i;
    };
    unsigned long long last = ~0ull;
    warp_union_pairs<NOUNION>(G, corner_pair ? ca : -1, cb, last);
    // Rounds: every lane turns up to kPairsPerLane of its events into slot
    // pairs in the warp's shared list; the list is then unioned with the pairs
    // spread over all 32 lanes (a lane with many events no longer serialises
    // the warp's union latency).
    while (__any_sync(kFull, ev | ne | nw)) {
        if (lane == 0) CCL_TASKSTAT(3, 1u);
        const int have = __popc(ev) + __popc(ne) + __popc(nw);
        const int take = min(have, kPairsPerLane);
        int incl = take;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int u = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += u;
        }
        const int total = __shfl_sync(kFull, incl, 31);
        const int pos = incl - take;
        int ia[kPairsPerLane], ib[kPairsPerLane];
#pragma unroll
        for (int e = 0; e < kPairsPerLane; ++e) {
            ia[e] = ib[e] = 0;
            if (e < take) {
                int x, xu;
                if (ev) {
                    x = (lane << 5) + __ffs(ev) - 1;
                    ev &= ev - 1;
                    xu = x;
                } else if (ne) {
                    x = (lane << 5) + __ffs(ne) - 1;
                    ne &= ne - 1;
                    xu = x + 1;
                } else {
                    x = (lane << 5) + __ffs(nw) - 1;
                    nw &= nw - 1;
                    xu = x - 1;
                }
                ia[e] = run_idx(0, x);
                ib[e] = run_idx(1, xu);
            }
        }
        // records of runs 0..31 of either row from the briefs (shuffles);
        // beyond that from the record lists (loads issued together)
        uint32_t va[kPairsPerLane], vb[kPairsPerLane];
#pragma unroll
        for (int e = 0; e < kPairsPerLane; ++e) {
            va[e] = __shfl_sync(kFull, r0, ia[e] & 31);
            vb[e] = __shfl_sync(kFull, rl, ib[e] & 31);
        }
#pragma unroll
        for (int e = 0; e < kPairsPerLane; ++e) {
            if (e < take && ia[e] >= kRL) va[e] = __ldcg(Rlo + ia[e]);
            if (e < take && ib[e] >= kRL) vb[e] = __ldcg(R + t_up * RCAP + up_base + ib[e]);
        }
#pragma unroll
        for (int e = 0; e < kPairsPerLane; ++e)
            if (e < take) pairs[pos + e] = make_int2(rec_slot(va[e], g.ntiles, t_lo), rec_slot(vb[e], g.ntiles, t_up));
        __syncwarp();
#ifdef CCL_K2_PHASES
        if (g_k2_phase && lane == 0 && g_k2_phase[4 * size_t(ptask) + 1] == 0) g_k2_phase[4 * size_t(ptask) + 1] = gtimer();
#endif
        for (int base = 0; base < total; base += 32) {
            const int i = base + lane;
            const int2 pr = i < total ? pairs[i] : make_int2(-1, -1);
            warp_union_pairs<NOUNION>(G, pr.x, pr.y, last);
#ifdef CCL_K2_PHASES
            __syncwarp();
            if (g_k2_phase && lane == 0 && g_k2_phase[4 * size_t(ptask) + 2] == 0) g_k2_phase[4 * size_t(ptask) + 2] = gtimer();
#endif
        }
        __syncwarp();
    }
    __syncwarp();
}

// The vertical boundary left of tile column bx >= 1 over kVBands = 32 / TY
// consecutive tile bands starting at band0: one warp, lane = row (all 32 lanes
// busy).  The NW / NE diagonal partners come from the lane above by shuffle;
// lane 0's (the corner of a horizontal boundary) is covered by boundary_h.
template <int TY>
__host__ __device__ constexpr int v_bands() { return 32 / TY; }

template <int TY, int CONN>
__device__ __forceinline__ void boundary_v(const Geom& g, const int32_t* E, uint64_t* G, int b, int band0,
                                           int bx) {
    const int lane = threadIdx.x & 31;
    const int band = band0 + lane / TY, r = lane % TY;
    uint64_t* Gb = G;  // edge slots are numbered over the whole batch
    int L = -1, Rr = -1;
    if (band < g.tiles_y && band * TY + r < g.H) {
        const int32_t* Er = E + tile_index(g, b, band, bx) * kEdgeCap;  // tile right of the edge
        const int32_t* El = Er - kEdgeCap;                               // tile left of the edge
        L = __ldcg(El + kEdgeRC + r);   // slot of the root of (x0-1, y), or -1
        Rr = __ldcg(Er + kEdgeLC + r);  // slot of the root of (x0, y), or -1
    }
    unsigned long long last = ~0ull;
    warp_union_pairs(Gb, (L >= 0 && Rr >= 0) ? L : -1, Rr, last);        // W edge of (x0, y)
    if (CONN == 8) {
        int Lu = __shfl_up_sync(kFull, L, 1), Ru = __shfl_up_sync(kFull, Rr, 1);
        if (lane == 0) Lu = Ru = -1;
        warp_union_pairs(Gb, (Rr >= 0 && Lu >= 0) ? Rr : -1, Lu, last);  // NW of (x0, y)
        warp_union_pairs(Gb, (L >= 0 && Ru >= 0) ? L : -1, Ru, last);    // NE of (x0-1, y)
    }
}

// K2 boundary analysis: one warp per horizontal tile boundary (1024 px) or per
// 32-row stretch of a vertical one; tasks are independent (lock-free unions).
template <int TY, int CONN, int DBG = 0>
#ifndef CCL_K2_MINB
#define CCL_K2_MINB 1  // min resident K2 blocks per SM (register cap: 65536 / (MINB * 32 * warps))
#endif
__global__ void __launch_bounds__(32 * kK2Warps, CCL_K2_MINB) k_boundary(Geom g, const uint32_t* __restrict__ bits,
                                                  const uint32_t* __restrict__ R,
                                                  const int32_t* __restrict__ E,
                                                  uint64_t* __restrict__ G, long long n_h, long long n_v,
                                                  int sub_log2 = 0) {
    __shared__ Word s_w[kK2Warps][2][kWords];
    __shared__ int2 s_pairs[kK2Warps][32 * kPairsPerLane];
    if (!g.epoch) pdl_wait();  // else: each task waits for its own tiles' ready flags
    const int warp = threadIdx.x >> 5;
    // (task counts are < 2^31: <= 2 per 16 x 1024 tile; 32-bit index math)
    const unsigned task = blockIdx.x * unsigned(kK2Warps) + unsigned(warp);
    if ((threadIdx.x & 31) == 0) CCL_TL_MIN(2);
    const unsigned long long t_start = (DBG & 8) ? gtimer() : 0ull;
    const unsigned nh_sub = unsigned(n_h) << sub_log2;  // horizontal boundaries, split in 2^sub_log2 warps each
    if (task < nh_sub) {
        if (DBG & 2) return;
        const unsigned th = task >> sub_log2;
        const unsigned q = g.div_tx.div(th);
        const int tx = int(th - q * unsigned(g.tiles_x));
        const unsigned q2 = g.div_ty1.div(q);
        const int band = 1 + int(q - q2 * unsigned(g.tiles_y - 1));
        const int b = int(q2);
        if (g.epoch) {  // the two tiles of the boundary and (8-conn corners) the upper tile's neighbours
            const int lane = threadIdx.x & 31;
            const size_t t_lo = tile_index(g, b, band, tx);
            if (lane == 0) wait_tile_ready(g, t_lo);
            if (lane == 1) wait_tile_ready(g, t_lo - g.tiles_x);
            if (CONN == 8 && lane == 2 && tx > 0) wait_tile_ready(g, t_lo - g.tiles_x - 1);
            if (CONN == 8 && lane == 3 && tx + 1 < g.tiles_x) wait_tile_ready(g, t_lo - g.tiles_x + 1);
            __syncwarp();
        }
        boundary_h<TY, CONN, (DBG & 4) != 0>(g, bits, R, E, G, b, band, tx, s_w[warp], s_pairs[warp],
                                             int(task & ((1u << sub_log2) - 1u)), sub_log2);
    } else if (task < nh_sub + unsigned(n_v)) {
        if (DBG & 1) return;
        const unsigned t = task - nh_sub;
        const unsigned q = g.div_tx1.div(t);
        const int bx = 1 + int(t - q * unsigned(g.tiles_x - 1));
        const unsigned q2 = g.div_vg.div(q);
        const unsigned groups = unsigned(g.tiles_y + v_bands<TY>() - 1) / v_bands<TY>();
        const int band0 = int(q - q2 * groups) * v_bands<TY>();
        const int b = int(q2);
        if (g.epoch) {  // the tiles left and right of the edge in each of the bands
            const int lane = threadIdx.x & 31, band = band0 + (lane >> 1);
            if (lane < 2 * v_bands<TY>() && band < g.tiles_y) wait_tile_ready(g, tile_index(g, b, band, bx - (lane & 1)));
            __syncwarp();
        }
        boundary_v<TY, CONN>(g, E, G, b, band0, bx);
    }
    if ((threadIdx.x & 31) == 0) CCL_TL_MAX(3);
    if ((DBG & 8) && (threadIdx.x & 31) == 0 && g_k2_stamps && task < nh_sub + unsigned(n_v)) {
        g_k2_stamps[2 * size_t(task)] = t_start;
        g_k2_stamps[2 * size_t(task) + 1] = gtimer();
    }
}

// ================================================================ K1 kernel
// Persistent: each block walks tiles t = blockIdx.x, +gridDim.x, ...; the
// 128-bit image loads of the NEXT tile are issued into registers before the
// current tile is processed, so HBM reads overlap the shared-memory work.
// (Fusing the boundary unions into this kernel -- each boundary merged by the
// block that publishes its second tile -- measured 4x slower: the blocks
// stall on the unions' global latency.)
template <int TY, int CONN, bool VEC, int DBG = 0, int THR = 0>
__global__ void __launch_bounds__(k1_threads<TY>(), k1_min_blocks<TY>()) k_local_merge(const uint8_t* __restrict__ img, Geom g,
                                                             uint32_t* __restrict__ bits,
                                                             uint64_t* __restrict__ G,
                                                             uint32_t* __restrict__ R,
                                                             int32_t* __restrict__ E,
                                                             int32_t* __restrict__ F,
                                                             unsigned ntiles) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K1Smem<TY>& sm = *reinterpret_cast<K1Smem<TY>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned t = blockIdx.x;
    // every K1 block is resident (persistent grid): the boundary analysis may
    // be scheduled onto the SM slots K1's finished blocks free (its tasks wait
    // on the per-tile ready flags)
    if (g.epoch) pdl_launch_dependents();
    if (threadIdx.x == 0) CCL_TL_MIN(0);
    if (t >= ntiles) return;
    constexpr bool PF = VEC;  // the first tile's register rows (k1_pf_rows)
    // one register set: loaded with tile t before the loop, then refilled with
    // the block's next tile as soon as the current one is in the masks
    // 256-bit image loads need 32-byte aligned rows
    const bool v8 = ((g.W & 31) == 0) && ((reinterpret_cast<uintptr_t>(img) & 31) == 0);
    ImgRegs<TY> a;
    if (PF) k1_prefetch<TY>(img, g, t, warp, lane, v8, a);
    if (threadIdx.x == 0) sm.ndefer = 0;
    // every tile whose runs fit the shared-memory lists is labelled as one
    // range; run-dense tiles are deferred to the loop below, so the range
    // machinery stays out of this loop's code and registers
    while (t < ntiles) {
        const int v = k1_masks<TY, CONN, VEC, false, DBG, THR>(sm, img, g, t, a, t + gridDim.x, ntiles, bits, warp, lane, v8);
        const bool fits = __shfl_sync(kFull, v, TY - 1) <= k1_cap<TY>();  // block-uniform
        if (fits) {
            k1_range<TY, CONN, DBG, true>(sm, g, t, decode_tile<TY>(g, t), v, 0, TY, 0, G, R, E, F, warp, lane);
        } else if (threadIdx.x == 0) {
            // (block b's list: g.defer[b * per ..], per = ceil(ntiles / grid) slots)
            g.defer[size_t(blockIdx.x) * ((ntiles + gridDim.x - 1) / gridDim.x) + sm.ndefer++] = t;
        }
        if (fits) k1_publish(g, t);
        t += gridDim.x;
    }
    __syncthreads();
    const int nd = sm.ndefer;
    for (int i = 0; i < nd; ++i) {
        const unsigned td = unsigned(__ldcg(g.defer + size_t(blockIdx.x) * ((ntiles + gridDim.x - 1) / gridDim.x) + i));
        const int v = k1_masks<TY, CONN, VEC, true, DBG, THR>(sm, img, g, td, a, ntiles, ntiles, bits, warp, lane, v8);
        k1_dense<TY, CONN, DBG>(sm, g, td, v, G, R, E, F, warp, lane);
        __syncthreads();  // smem is reused by the next deferred tile
    }
    if (threadIdx.x == 0) CCL_TL_MAX(1);
}

// ------------------------------------------- K2 tail: resolve edge roots
// Boundary analysis, last step: every edge-touching local root of every tile
// is resolved to its global root (find) once, all in parallel,
// and 1 + root is stored in the tile's F list, so K3 needs no pointer chasing.
//
// Every edge root is owned by exactly one resolving thread (it is a local root
// of one tile), and the long chains of the forest consist of edge roots only,
// so the threads do concurrent pointer jumping: each repeatedly re-points ITS
// node at the grandparent it reads (L2-coherent loads).  Other threads walking
// through that node then skip ahead, so a chain of depth d is resolved in
// ~log d rounds instead of d dependent loads (the read-only walk left the
// kernel waiting on a few 30+-hop chains).  Entries only ever move to
// ancestors, so the forest stays valid for later readers.
// Root entry (X << 32 | root) of edge slot s, with pointer jumping on s's own
// entry (re-pointed at each grandparent read; only ancestors are ever stored).
__device__ __forceinline__ uint64_t resolve_slot(uint64_t* G, unsigned s) {
    uint64_t v = __ldcg(reinterpret_cast<const unsigned long long*>(G) + s);
    if (unsigned(v) == s) return v;
    CCL_LOOP_GUARD(pj);
    while (true) {
        CCL_LOOP_TICK(pj);
        const uint64_t w = __ldcg(reinterpret_cast<const unsigned long long*>(G) + unsigned(v));
        if (unsigned(w) == unsigned(v)) return w;  // v's parent is the root: w is the root's entry
        CCL_ASSERT((w >> 32) < (v >> 32));
        __stcg(reinterpret_cast<unsigned long long*>(G) + s, static_cast<unsigned long long>(w));
        v = w;
    }
}

template <int TY>
__global__ void __launch_bounds__(256) k_resolve(Geom g, uint64_t* __restrict__ G,
                                                 const int32_t* __restrict__ E,
                                                 int32_t* __restrict__ F, unsigned ntiles) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (unsigned t = (blockIdx.x * 256u + threadIdx.x) >> 5; t < ntiles; t += (gridDim.x * 256u) >> 5) {
        const int n = E[size_t(t) * kEdgeCap];
        for (int i = lane; i < n; i += 32) {
            const unsigned s = edge_slot(g.ntiles, i, t);
            F[s] = int(resolve_slot(G, s) >> 32) + 1 + g.label_off;
        }
    }
}

// Strip mode (ccl_strip.cuh): the final label of an edge root on a strip
// boundary row is the minimum label of its slot set in the slot union-find.
struct StripFinal {
    const int32_t* F;         // F[root slot] = INT_MAX - its first boundary slot, or -1
    uint64_t* P;              // slot union-find over the k * 2W boundary slots
    const int32_t* gathered;  // all ranks' send buffers (labels, reps)
    int W, slot0;             // slot0 = this rank's first slot (rank * 2W)
};
__device__ __forceinline__ uint64_t slot_find(uint64_t* P, const int32_t* gathered, int W, unsigned s);

// Final label of edge root i of tile t: its root in G (pointer jumping), and
// in strip mode (!RES) for a root on a strip boundary the slot set's minimum.
template <bool RES>
__device__ __forceinline__ int edge_label(const Geom& g, uint64_t* G, const StripFinal& sf, unsigned t, int i) {
    const uint64_t w = resolve_slot(G, edge_slot(g.ntiles, i, t));
    int lab = int(w >> 32) + 1 + g.label_off;
    if (!RES) {
        const int v = __ldcg(sf.F + unsigned(w));
#ifdef CCL_CHECK
        if (v < -1 || (v >= 0 && INT_MAX - v >= 2 * sf.W))
            printf("edge_label: tile %u edge %d root entry %llx F %d\n", t, i, (unsigned long long)w, v);
#endif
        CCL_ASSERT(v == -1 || (v >= 0 && INT_MAX - v < 2 * sf.W));
        if (v >= 0) lab = int(slot_find(sf.P, sf.gathered, sf.W, unsigned(sf.slot0 + (INT_MAX - v))) >> 32);
    }
    return lab;
}

// The helper warp's shared slot holds the first kFlCap edge labels of a tile
// (texture tiles use a few tens; only tiles labelled in several row ranges
// exceed it -- the label table resolves those few entries itself).
#ifndef CCL_K3_TAILSYNC
#define CCL_K3_TAILSYNC 0  // a barrier after each tile's last window as well (0.37 us/step slower)
#endif
#ifndef CCL_K3_TU
#define CCL_K3_TU 4  // K3 label table: runs per thread and iteration (noise K3 137 -> 92 us; texture unchanged)
#endif
constexpr int kK3TU = CCL_K3_TU;
#ifndef CCL_K3_FLCAP
#define CCL_K3_FLCAP 1088
#endif
constexpr int kFlCap = CCL_K3_FLCAP;

// ================================================================ K3: link
// Final link (§2.3).  Per tile:
//  1. row runs re-derived from the bit mask (run numbering only, no
//     union-find);
//  2. one thread per run: final label = 1 + global root (K1's per-run record),
//     or the boundary analysis' resolved label when the component touches a
//     tile edge -> label table lab[run id];
//  3. per tile row, every lane expands its own 32-px word into labels
//     (branch-free, 4-px groups) into a per-warp shared-memory row buffer in
//     the TMA 128-byte-swizzle layout, and one lane issues a bulk-tensor store
//     of the 4 KB row.
// The label table holds kLabCap runs; a tile with more runs (noise-like
// content) is linked in row windows that each fit the table (54 KB of shared
// memory per block).  3 blocks per SM: 4 (register-capped at 64) measured
// 57 vs 54 us on C3 texture -- more concurrent row streams, lower DRAM
// efficiency -- though faster on noise (121 vs 150 us); 2 and 1: 62 / 90 us.
// Persistent like K1: the next tile's mask words, first run records and first
// resolved labels are prefetched into registers while the current tile is
// processed.
constexpr int kLabCap = 4096;

struct __align__(8) LWord {
    uint32_t m;   // foreground mask
    int32_t pad;  // run starts in the row before this word
};

template <int TY>
struct __align__(1024) LinkSmem {
    // per-warp row of labels, two 2-KB halves in the TMA SWIZZLE_64B layout
    // (CCL_K3_HALF; pixels 0-15 / 16-31 of every 32-px word, see tma_store_half),
    // else one SWIZZLE_128B box (16-B unit q of word w at w*128 + ((q ^ (w & 7)) * 16));
    // both conflict-free for the lanes
    int4 rowbuf[kWarps][kTileW / 4];
    LWord wd[TY][kWords];
    int32_t lab[kLabCap];            // final label of tile run k (current row window)
    uint4 rc[kRunCache / 4];         // first run records of the tile (prefetched)
    int32_t fl[2][kFlCap];           // final labels of the edge roots i < kFlCap of tiles j, j+1 (helper warp)
    int32_t produced;                // tiles whose fl slot the helper warp has filled
    int32_t consumed;                // tiles whose fl slot the compute warps are done with
    int32_t rcnt[TY];
    int32_t rbase[TY + 1];
};

template <int TY>
struct LinkRegs {
    uint32_t m[TY / kWarps];
    uint4 runs;  // warps w < kRunCache / 128: run records 4*i .. 4*i+3 (i = 32 * w + lane)
};

template <int TY>
__device__ __forceinline__ void k3_prefetch(const uint32_t* bits, const uint32_t* R,
                                            const Geom& g, unsigned t, int warp, int lane,
                                            LinkRegs<TY>& pf) {
    const TileId id = decode_tile<TY>(g, t);
    const uint32_t* bm = bits + size_t(id.b) * size_t(g.nwords);
    const int wg = id.tx * kWords + lane;
#pragma unroll
    for (int i = 0; i < TY / kWarps; ++i) {
        const int y = id.y0 + warp + i * kWarps;
        pf.m[i] = (y < g.H && wg < g.WW) ? __ldg(bm + size_t(y) * g.WW + wg) : 0u;
    }
    if (warp < kRunCache / 128)
        pf.runs = __ldg(reinterpret_cast<const uint4*>(R + size_t(t) * runs_per_tile_cap<TY>()) + lane + 32 * warp);
}

// TMA bulk-tensor store of one 1024-px label row from shared memory: the
// labels tensor is viewed as [rows][W/32][32] int32, the box is [1][32][32]
// (out-of-range chunks of the last tile column are clipped by the hardware).
__device__ __forceinline__ void tma_store_row(const CUtensorMap* tmap, const void* smem, int chunk0, int row) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                 ::"l"(reinterpret_cast<uint64_t>(tmap)), "r"(0), "r"(chunk0), "r"(row), "r"(sa)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// CCL_K3_HALF: a row leaves as two half-row stores (pixels 0-15 / 16-31 of
// every 32-px word: box [1][32][16], SWIZZLE_64B -- 16-B unit q of word w at
// w*64 + ((q ^ ((w >> 1) & 3)) * 16)), so the wait for the previous row's
// half to have been read overlaps the other half's expansion.
#ifndef CCL_K3_SPLIT
#define CCL_K3_SPLIT 2  // stores per row: 1 (SWIZZLE_128B), 2 (64B) or 4 (32B)
#endif
#define CCL_K3_HALF (CCL_K3_SPLIT > 1)
__device__ __forceinline__ void tma_store_half(const CUtensorMap* tmap, const void* smem, int px0, int chunk0, int row) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                 ::"l"(reinterpret_cast<uint64_t>(tmap)), "r"(px0), "r"(chunk0), "r"(row), "r"(sa)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// all but the newest SPLIT - 1 bulk groups have read their shared memory
__device__ __forceinline__ void tma_wait_read_but1() {
    if (CCL_K3_SPLIT == 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// x | all lower bits of x within each 4-bit nibble (prefix OR per nibble)
__device__ __forceinline__ uint32_t nibble_prefix_or(uint32_t x) {
    x |= (x << 1) & 0xEEEEEEEEu;
    return x | ((x << 2) & 0xCCCCCCCCu);
}

// x != 0 ? a : b as a predicated select (keeps the expansion loop branch-free)
__device__ __forceinline__ int selp_nz(uint32_t x, int a, int b) {
    int r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.b32 %0, %1, %2, q;\n\t}"
        : "=r"(r) : "r"(a), "r"(b), "r"(x));
    return r;
}

// 16-byte slot of 4-px group q (0..255) of a row in the swizzled row buffer:
// group q = 8*w + g (word w, group g within the word) lives at 8*w + (g ^ (w & 7)).
__device__ __forceinline__ int swz(int w, int g) { return (w << 3) + (g ^ (w & 7)); }

template <int TY, int CONN, bool VEC, bool TMA, bool RES, int DBG = 0>
__device__ __forceinline__ void k3_tile(LinkSmem<TY>& sm, const Geom& g, const uint32_t* bits, unsigned t, int j,
                                        const LinkRegs<TY>& cur, const uint32_t* R, int32_t* out,
                                        const CUtensorMap* tmap, int warp, int lane, uint64_t* G,
                                        const StripFinal& sf) {
    const TileId id = decode_tile<TY>(g, t);
    int32_t* ob = out + size_t(id.b) * size_t(g.npx);
    const uint32_t* Rt = R + size_t(t) * runs_per_tile_cap<TY>();
    const int32_t* Fl = sm.fl[j & 1];
    const int tid = threadIdx.x;
    if ((DBG & 4) && threadIdx.x == 0) k3_stamp(t, 0);

    if (warp < kRunCache / 128) sm.rc[lane + 32 * warp] = cur.runs;
    if (tid == 0) {  // the helper warp has this tile's edge labels in slot j & 1
        while (ld_volatile(&sm.produced) <= j) __nanosleep(32);
    }
    // 1. run starts and run numbering of every row
#pragma unroll
    for (int i = 0; i < TY / kWarps; ++i) {
        const int r = warp + i * kWarps;
        const uint32_t m = cur.m[i];
        uint32_t pm = __shfl_up_sync(kFull, m, 1);
        if (lane == 0) pm = 0;
        const uint32_t s = m & ~((m << 1) | (pm >> 31));
        const int n = __popc(s);
        int incl = n;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int u = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += u;
        }
        sm.wd[r][lane] = LWord{m, incl - n};
        if (lane == 31) sm.rcnt[r] = incl;
    }
    k3_sync();
    if ((DBG & 4) && threadIdx.x == 0) k3_stamp(t, 1);
    // run base of every row (lane r of every warp: v = first run id of row r+1)
    int v = lane < TY ? sm.rcnt[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(kFull, v, d);
        if (lane >= d) v += u;
    }
    if (warp == 0 && lane < TY) sm.rbase[lane + 1] = v;
    if (warp == 0 && lane == 0) sm.rbase[0] = 0;
    const int W = g.W, x0 = id.x0, y0 = id.y0;
    int4* buf = sm.rowbuf[warp];
    // row windows [r0, r1) whose runs fit the label table (one window unless
    // the tile has more than kLabCap runs)
    int r0 = 0;
    while (r0 < TY) {  // block-uniform
        const int base = r0 > 0 ? __shfl_sync(kFull, v, r0 - 1) : 0;
        const unsigned fit = __ballot_sync(kFull, lane >= r0 && lane < TY && v - base <= kLabCap);
        const int r1 = 32 - __clz(fit);  // rows r0 .. r1-1 (v is monotone; >= 1 row: <= 512 runs per row)
        const int end = __shfl_sync(kFull, v, r1 - 1);
        // 2. label table, one thread per run of the window (CCL_K3_TU runs per
        // thread and iteration: their record loads in flight together)
#pragma unroll 1
        for (int k0 = base + tid; k0 < end; k0 += kK3TU * kThreads) {
            uint32_t rec[kK3TU];
#pragma unroll
            for (int u = 0; u < kK3TU; ++u) {
                const int k = k0 + u * kThreads;
                rec[u] = k >= end ? 0u : (k < kRunCache ? reinterpret_cast<const uint32_t*>(sm.rc)[k] : __ldg(Rt + k));
            }
#pragma unroll
            for (int u = 0; u < kK3TU; ++u) {
                const int k = k0 + u * kThreads;
                if (k >= end) break;
                const int e = int(rec[u] >> 16);  // 1 + edge-list index, or 0
                const int rr = int(rec[u] & 0x7FFFu);
                int lab = (y0 + (rr >> 10)) * W + x0 + (rr & 1023) + 1 + g.label_off;
                if (e) lab = e <= kFlCap ? Fl[e - 1] : edge_label<RES>(g, G, sf, t, e - 1);
                sm.lab[k - base] = lab;
            }
        }
        k3_sync();
        if ((DBG & 4) && threadIdx.x == 0) k3_stamp(t, 2);

        // 3. expand and stream the window's rows
        for (int r = r0 + warp; r < r1; r += kWarps) {
            const int y = y0 + r;
            if (y >= g.H) break;
            int32_t* orow = ob + size_t(y) * size_t(W) + x0;
            const int rb = sm.rbase[r] - base;
            if (VEC) {
                if (TMA) {  // the previous row's bulk store (CCL_K3_HALF: its first half) must have read the buffer
                    if (lane == 0) {
                        if (CCL_K3_HALF) tma_wait_read_but1();
                        else tma_wait_read_all();
                    }
                    __syncwarp();
                }
                const LWord wd = sm.wd[r][lane];
                const uint32_t m = wd.m;
                uint32_t pm = __shfl_up_sync(kFull, m, 1);
                if (lane == 0) pm = 0;
                const uint32_t s = m & ~((m << 1) | (pm >> 31));
                int idx = rb + wd.pad - 1;           // run covering the word's bit 0 (if fg, not a start)
                int c = ((m & 1u) && !(s & 1u)) ? sm.lab[idx] : 0;
                const int lim = end - base - 1;      // last valid table entry (guards the speculative loads)
                // A 4-px group holds at most two run starts (starts are never
                // adjacent), so each pixel's label is 0, c (the run entering the
                // group), L1 or L2 (the group's first / second new run).  2-bit
                // code per pixel, built for the whole word at once: P1 / P2 = "at
                // least one / two starts at or before this pixel within its group".
                const uint32_t P1 = nibble_prefix_or(s);
                const uint32_t P2 = nibble_prefix_or(s & ((P1 << 1) & 0xEEEEEEEEu));
                const uint32_t Hi = m & P1;           // code 2 (L1) or 3 (L2)
                const uint32_t Lo = m & (~P1 | P2);   // code 1 (c) or 3 (L2)
#pragma unroll
                for (int q = 0; q < (DBG & 1 ? 0 : 8); ++q) {
                    constexpr int QP = 8 / CCL_K3_SPLIT;  // 4-px groups per part
                    if (TMA && CCL_K3_HALF && q > 0 && q % QP == 0) {  // part out; the previous row's next part read
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_half(tmap, buf + (q / QP - 1) * (256 / CCL_K3_SPLIT), (q / QP - 1) * (32 / CCL_K3_SPLIT),
                                           x0 >> 5, id.b * g.H + y);
                            tma_wait_read_but1();
                        }
                        __syncwarp();
                    }
                    const int L1 = sm.lab[min(idx + 1, lim)], L2 = sm.lab[min(idx + 2, lim)];
                    int px[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t bit = 1u << (4 * q + j);
                        px[j] = selp_nz(Hi & bit, selp_nz(Lo & bit, L2, L1), selp_nz(Lo & bit, c, 0));
                    }
                    if (TMA && CCL_K3_SPLIT == 2)
                        buf[(q >> 2) * 128 + lane * 4 + ((q & 3) ^ ((lane >> 1) & 3))] = make_int4(px[0], px[1], px[2], px[3]);
                    else if (TMA && CCL_K3_SPLIT == 4)  // SWIZZLE_32B: unit u of word w at w*32 + ((u ^ ((w >> 2) & 1)) * 16)
                        buf[(q >> 1) * 64 + lane * 2 + ((q & 1) ^ ((lane >> 2) & 1))] = make_int4(px[0], px[1], px[2], px[3]);
                    else
                        buf[swz(lane, q)] = make_int4(px[0], px[1], px[2], px[3]);
                    c = px[3];  // pixel 3 background => the next fg pixel starts a run
                    idx += __popc((s >> (4 * q)) & 0xFu);
                }
                if (TMA) {
                    fence_proxy_async_smem();  // generic-proxy smem writes -> async proxy
                    __syncwarp();
                    if (lane == 0) {
                        if (CCL_K3_HALF)
                            tma_store_half(tmap, buf + (CCL_K3_SPLIT - 1) * (256 / CCL_K3_SPLIT),
                                           (CCL_K3_SPLIT - 1) * (32 / CCL_K3_SPLIT), x0 >> 5, id.b * g.H + y);
                        else tma_store_row(tmap, buf, x0 >> 5, id.b * g.H + y);
                    }
                } else {
                    __syncwarp();
#pragma unroll 2
                    for (int j = 0; j < kTileW / 128; ++j) {
                        const int x = 128 * j + 4 * lane;
                        if (x0 + x >= W) break;
                        const int4 o = buf[swz(4 * j + (lane >> 3), lane & 7)];
                        st_stream_i4(orow + x, o.x, o.y, o.z, o.w);
                    }
                    __syncwarp();
                }
            } else {
                // generic widths: lane writes pixel (k<<5) + lane of every word k
                for (int k = 0; k < kWords; ++k) {
                    const int x = (k << 5) + lane;
                    if (x0 + x < W) {
                        const LWord wd = sm.wd[r][k];
                        const uint32_t pm = k > 0 ? sm.wd[r][k - 1].m : 0u;
                        const uint32_t s = wd.m & ~((wd.m << 1) | (pm >> 31));
                        int o = 0;
                        if ((wd.m >> lane) & 1u) o = sm.lab[rb + wd.pad + __popc(s & (kFull >> (31 - lane))) - 1];
                        orow[x] = o;
                    }
                }
            }
        }
        r0 = r1;
        // the next window's table overwrites lab; after the tile's last window
        // no barrier: each warp's next-tile writes (its own rows' words, the
        // record cache) touch nothing another warp's expansion still reads, and
        // the next tile's first barrier orders everything else
        if (CCL_K3_TAILSYNC || r0 < TY) k3_sync();
    }
#ifndef CCL_K3_DISCARD
#define CCL_K3_DISCARD 1
#endif
#if CCL_K1_KEEP && CCL_K3_DISCARD
    // K1's mask rows and run records of this tile have had their last reader:
    // drop their (evict_last, dirty) L2 lines without a DRAM write-back.  Only
    // whole 128-byte lines owned by this tile (mask rows when W % 1024 == 0).
    {
        const int total = __shfl_sync(kFull, v, TY - 1);
        for (int i = tid; i < (total + 31) / 32; i += kThreads) l2_discard(Rt + 32 * i);
        if ((W & 1023) == 0 && lane < TY / kWarps) {
            const int y = y0 + warp + lane * kWarps;
            if (y < g.H)
                l2_discard(bits + size_t(id.b) * size_t(g.nwords) + size_t(y) * g.WW + id.tx * kWords);
        }
    }
#endif
    if (tid == 0) *reinterpret_cast<volatile int32_t*>(&sm.consumed) = j + 1;  // slot j & 1 is free again
    if ((DBG & 4) && threadIdx.x == 0) k3_stamp(t, 3);
}

// K3's helper warp (warp 8): the final labels of each of the block's tiles'
// edge roots, one tile ahead of the compute warps, into the shared slot
// j & 1.  RES: resolved here from the parent forest (the boundary analysis'
// resolve step, moved off its own launch into K3's bandwidth-bound shadow):
// concurrent pointer jumping -- every edge root is owned by exactly one
// thread, which keeps re-pointing its own entry at the grandparent it reads,
// so chains shared by many roots collapse in ~log d rounds; entries only ever
// move to ancestors.  !RES (strip mode): copy the labels the strip stages left
// in F.  k3_resolve_tile does one tile's roots i = first, first + stride, ...
constexpr int kK3Threads = kThreads + 32;  // 8 compute warps + the helper warp


template <bool RES>
__device__ __forceinline__ void k3_resolve_tile(int32_t* slot, const Geom& g, const int32_t* E, uint64_t* G,
                                                const StripFinal& sf, unsigned t, int first, int stride) {
    const int n = min(__ldcg(E + size_t(t) * kEdgeCap), kFlCap);
#ifdef CCL_K3_NORES  // timing experiments only: no resolve (wrong labels)
    for (int i = first; i < n; i += stride) slot[i] = i;
#else
    for (int i = first; i < n; i += stride) slot[i] = edge_label<RES>(g, G, sf, t, i);
#endif
}

#ifndef CCL_K3_COOP
#define CCL_K3_COOP 1
#endif

// The helper warp's loop over the block's tiles j0, j0+1, ... (t = blockIdx.x
// + j * gridDim.x).
template <int TY, bool RES>
__device__ __forceinline__ void k3_helper(LinkSmem<TY>& sm, const Geom& g, const int32_t* E, uint64_t* G,
                                          const StripFinal& F, unsigned ntiles, int j0) {
    const int lane = threadIdx.x & 31;
    int j = j0;
    for (unsigned t = blockIdx.x + unsigned(j0) * gridDim.x; t < ntiles; t += gridDim.x, ++j) {
        if (lane == 0) {  // slot j & 1 was last used by tile j - 2
            while (ld_volatile(&sm.consumed) < j - 1) __nanosleep(64);
        }
        __syncwarp();
        k3_resolve_tile<RES>(sm.fl[j & 1], g, E, G, F, t, lane, 32);
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            *reinterpret_cast<volatile int32_t*>(&sm.produced) = j + 1;
        }
    }
}


template <int TY, int CONN, bool VEC, bool TMA = false, bool RES = true, int DBG = 0>
__global__ void __launch_bounds__(kK3Threads, 3) k_link(Geom g, const uint32_t* __restrict__ bits,
                                                        const uint32_t* __restrict__ R,
                                                        const int32_t* __restrict__ E,
                                                        uint64_t* __restrict__ G,
                                                        const StripFinal F,
                                                        int32_t* __restrict__ out, unsigned ntiles,
                                                        const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    LinkSmem<TY>& sm = *reinterpret_cast<LinkSmem<TY>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) CCL_TL_MIN(4);
    if (threadIdx.x == 0) {
        sm.produced = 0;
        sm.consumed = 0;
    }
    __syncthreads();
    unsigned t = blockIdx.x;
    if (t >= ntiles) return;
    // The mask words and run records are K1's outputs, complete before the
    // boundary analysis started: the compute warps load their first two tiles'
    // share BEFORE waiting for the boundary analysis to finish (under PDL this
    // block is already resident while it drains).
    LinkRegs<TY> a, b;
    if (warp < kWarps && g.k3_early) {
        k3_prefetch<TY>(bits, R, g, t, warp, lane, a);
        if (t + gridDim.x < ntiles) k3_prefetch<TY>(bits, R, g, t + gridDim.x, warp, lane, b);
    }
    pdl_wait();
    if (threadIdx.x == 0) CCL_TL_MIN(5);
    if (warp < kWarps && !g.k3_early) {  // K3 right after K1 (no boundaries): K1's outputs only after the wait
        k3_prefetch<TY>(bits, R, g, t, warp, lane, a);
        if (t + gridDim.x < ntiles) k3_prefetch<TY>(bits, R, g, t + gridDim.x, warp, lane, b);
    }
    // The block's first tile: all 9 warps resolve its edge roots together
    // (one chain latency instead of n / 32 of them on the helper alone -- the
    // compute warps would otherwise wait for it); the helper takes the rest.
    int j0 = 0;
    if (CCL_K3_COOP) {
        k3_resolve_tile<RES>(sm.fl[0], g, E, G, F, t, threadIdx.x, kK3Threads);
        __syncthreads();
        if (threadIdx.x == 0) sm.produced = 1;
        j0 = 1;
    }
    if (warp == kWarps) {
        k3_helper<TY, RES>(sm, g, E, G, F, ntiles, j0);
        return;
    }
    int j = 0;
    while (true) {
        if (j > 0 && t + gridDim.x < ntiles) k3_prefetch<TY>(bits, R, g, t + gridDim.x, warp, lane, b);
        k3_tile<TY, CONN, VEC, TMA, RES, DBG>(sm, g, bits, t, j++, a, R, out, &tmap, warp, lane, G, F);
        t += gridDim.x;
        if (t >= ntiles) break;
        if (t + gridDim.x < ntiles) k3_prefetch<TY>(bits, R, g, t + gridDim.x, warp, lane, a);
        k3_tile<TY, CONN, VEC, TMA, RES, DBG>(sm, g, bits, t, j++, b, R, out, &tmap, warp, lane, G, F);
        t += gridDim.x;
        if (t >= ntiles) break;
    }
    if (TMA && lane == 0) tma_wait_all();  // smem must outlive the bulk stores
    if (threadIdx.x == 0) CCL_TL_MAX(6);
}

}  // namespace ccl
