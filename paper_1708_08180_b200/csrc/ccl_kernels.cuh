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
#include <cstdint>
#include <cuda_runtime.h>

namespace ccl {

constexpr int kTileW = 1024;   // pixels per tile row
constexpr int kWords = 32;     // 32-bit mask words per tile row
constexpr int kThreads = 256;  // threads per K1/K3 block
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kTag = int(0x80000000u);

struct Geom {
    int B, H, W;       // batch, rows, columns
    int WW;            // mask words per image row = ceil(W/32)
    int tiles_x;       // ceil(W/1024)
    int tiles_y;       // ceil(H/TY)
    long long npx;     // H*W  (per image)
    long long nwords;  // H*WW (per image)
};

// One 32-px mask word with its row-run description (one 128-bit smem load).
struct __align__(16) Word {
    uint32_t m;  // foreground mask
    uint32_t s;  // run-start mask (tile-local runs)
    int32_t c;   // x (0..1023) of the run start owning bit 0 of the word (if fg), else -1
    int32_t pad;
};

// Shared-memory layout of one K1/K3 tile (dynamic shared memory).
template <int TY>
struct TileSmem {
    Word wd[TY][kWords];        // .pad = row-local index of the word's first run
    int32_t P[TY * kTileW / 2]; // parent: index (l>>1), value = tile-local index l of parent
    uint32_t flag[TY * kTileW / 64];  // "root touches a tile edge" bits, index (l>>1)
    int32_t rcnt[TY];           // runs per tile row
};

// Per-run record written by K1 and read by K3 (uint16 per run, runs of a tile
// in raster order of their starts): bits 0..14 = tile-local index of the run's
// local root, bit 15 = that root's component touches a tile edge (so its final
// label must be resolved through the global parent array G).
constexpr int kRunEdgeBit = 0x8000;
template <int TY>
__host__ __device__ constexpr int runs_per_tile_cap() { return TY * kTileW / 2; }

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t nz4(uint32_t w) {
    // 4-bit mask of the nonzero bytes of w
    uint32_t t = (((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u;
    return ((t >> 7) * 0x00204081u >> 21) & 0xFu;
}

__device__ __forceinline__ uint32_t nz16(uint4 v) {
    return nz4(v.x) | (nz4(v.y) << 4) | (nz4(v.z) << 8) | (nz4(v.w) << 12);
}

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

// ----------------------------------------------- shared-memory union-find
// find / merge of §2.1.3 over tile-local run-start indices.
// Path halving: every visited node is re-pointed at its grandparent (an
// ancestor, so set membership never changes; values only move toward roots).
__device__ __forceinline__ int find_s(int32_t* P, int a) {
    volatile int32_t* V = P;
    int p = V[a >> 1];
    while (p != a) {
        const int gp = V[p >> 1];
        if (gp != p) V[a >> 1] = gp;
        a = p;
        p = gp;
    }
    return a;
}

// Read-only find: used by the flatten phase, which must leave every run start
// pointing at its root (a concurrent halving store could otherwise overwrite a
// flattened entry with a non-root ancestor).
__device__ __forceinline__ int find_s_ro(const int32_t* P, int a) {
    const volatile int32_t* V = P;
    int p = V[a >> 1];
    while (p != a) {
        a = p;
        p = V[a >> 1];
    }
    return a;
}

// Lock-free minimum-root union (reading R11): the larger root is re-pointed at
// the smaller with atomicMin; if someone else re-linked it first, retry with
// the value it was linked to.
__device__ __forceinline__ void union_s(int32_t* P, int a, int b) {
    while (true) {
        a = find_s(P, a);
        b = find_s(P, b);
        if (a == b) return;
        if (a < b) { int t = a; a = b; b = t; }
        const int old = atomicMin(&P[a >> 1], b);
        if (old == a) return;
        a = old;
    }
}

// -------------------------------------------------- global union-find (K2)
__device__ __forceinline__ void st_volatile(int32_t* p, int v) {
    *reinterpret_cast<volatile int32_t*>(p) = v;
}

// find with path halving in global memory (safe under concurrent min-unions:
// a halving store writes an ancestor of a non-root node, R11).
__device__ __forceinline__ int find_g(int32_t* G, int a) {
    int p = ld_volatile(G + a);
    while (p != a) {
        const int gp = ld_volatile(G + p);
        if (gp != p) st_volatile(G + a, gp);
        a = p;
        p = gp;
    }
    return a;
}

__device__ __forceinline__ void union_g(int32_t* G, int a, int b) {
    while (true) {
        a = find_g(G, a);
        b = find_g(G, b);
        if (a == b) return;
        if (a < b) { int t = a; a = b; b = t; }
        const int old = atomicMin(G + a, b);
        if (old == a) return;
        a = old;
    }
}

// ------------------------------------------------------------- tile decode
struct TileId {
    int b, tx, ty, x0, y0;
};

template <int TY>
__device__ __forceinline__ TileId decode_tile(const Geom& g, unsigned t) {
    TileId id;
    const unsigned q = t / unsigned(g.tiles_x);
    id.tx = int(t - q * unsigned(g.tiles_x));
    const unsigned q2 = q / unsigned(g.tiles_y);
    id.ty = int(q - q2 * unsigned(g.tiles_y));
    id.b = int(q2);
    id.x0 = id.tx * kTileW;
    id.y0 = id.ty * TY;
    return id;
}

// ------------------------------------------- K1 / K3 shared local labeling
// Phase L1: masks -> smem, run starts, carries, parent init.  `m` is this
// lane's mask word of tile row r.
template <int TY, bool INIT_P>
__device__ __forceinline__ void tile_row_init(TileSmem<TY>& sm, int r, int lane, uint32_t m) {
    uint32_t s;
    int c;
    row_runs(m, lane, s, c);
    // row-local run index of this word's first run start (exclusive prefix)
    const int n = __popc(s);
    int incl = n;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += t;
    }
    Word wd;
    wd.m = m;
    wd.s = s;
    wd.c = c;
    wd.pad = incl - n;
    sm.wd[r][lane] = wd;
    if (lane == 31) sm.rcnt[r] = incl;
    if (INIT_P) {
        const int base = r * kTileW + (lane << 5);
        uint32_t t = s;
        while (t) {
            const int bit = __ffs(t) - 1;
            t &= t - 1;
            const int l = base + bit;
            sm.P[l >> 1] = l;
        }
    }
}

// Tile-local index of the first run of tile row r (prefix of rcnt; after a
// barrier that follows tile_row_init of all rows).
template <int TY>
__device__ __forceinline__ int row_run_base(const TileSmem<TY>& sm, int r, int lane) {
    int v = lane < TY ? sm.rcnt[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(kFull, v, d);
        if (lane >= d) v += t;
    }
    const int incl = __shfl_sync(kFull, v, r > 0 ? r - 1 : 0);
    return r > 0 ? incl : 0;
}

// Every adjacency between a run of tile row r and a run of row r-1 yields one
// event f(cs, us) (cs, us = tile-local indices of the two run starts): the
// start of each overlap segment (4-conn, Alg. 1 l.14-18 / l.27-29 at run
// granularity) plus, for 8-conn, the diagonal run contacts NE / NW that do not
// overlap (reading R2/R10).  Out-of-tile neighbours count as background.
template <int TY, int CONN, typename F>
__device__ __forceinline__ void for_each_row_event(const TileSmem<TY>& sm, int r, int lane, F f) {
    const uint32_t cur = sm.wd[r][lane].m, up = sm.wd[r - 1][lane].m;
    uint32_t curL = __shfl_up_sync(kFull, cur, 1), upL = __shfl_up_sync(kFull, up, 1);
    uint32_t curR = __shfl_down_sync(kFull, cur, 1), upR = __shfl_down_sync(kFull, up, 1);
    if (lane == 0) { curL = 0; upL = 0; }
    if (lane == 31) { curR = 0; upR = 0; }
    const uint32_t o = cur & up, oL = curL & upL;
    uint32_t ev = o & ~((o << 1) | (oL >> 31));  // overlap-segment starts
    const int rb = r * kTileW, ub = (r - 1) * kTileW, xb = lane << 5;
    const Word* wc = sm.wd[r];
    const Word* wu = sm.wd[r - 1];
    while (ev) {
        const int x = xb + __ffs(ev) - 1;
        ev &= ev - 1;
        f(rb + run_start_x(wc, x), ub + run_start_x(wu, x));
    }
    if (CONN == 8) {
        const uint32_t cur_n = (cur >> 1) | (curR << 31), up_n = (up >> 1) | (upR << 31);
        const uint32_t cur_p = (cur << 1) | (curL >> 31), up_p = (up << 1) | (upL >> 31);
        uint32_t ne = cur & ~cur_n & ~up & up_n;  // upper run starts at x+1
        uint32_t nw = cur & ~cur_p & ~up & up_p;  // current run starts at x, upper ends at x-1
        while (ne) {
            const int x = xb + __ffs(ne) - 1;
            ne &= ne - 1;
            f(rb + run_start_x(wc, x), ub + x + 1);
        }
        while (nw) {
            const int x = xb + __ffs(nw) - 1;
            nw &= nw - 1;
            f(rb + x, ub + run_start_x(wu, x - 1));
        }
    }
}

// Calls f(l) for every run start l of tile row r held by this lane.
template <int TY, typename F>
__device__ __forceinline__ void for_each_run_start(const TileSmem<TY>& sm, int r, int lane, F f) {
    uint32_t t = sm.wd[r][lane].s;
    const int base = r * kTileW + (lane << 5);
    while (t) {
        const int bit = __ffs(t) - 1;
        t &= t - 1;
        f(base + bit);
    }
}

// Local merge of one tile whose masks / runs / P are initialised in smem.
// Coarse labeling: the row scan + row unification of Alg. 1 (l.9-13, l.19-24
// in the row direction) is exact here -- every pixel's provisional label is
// its run start, the lowest equivalent label of its row segment.
// COARSE_COLUMN additionally performs the column scan (l.14-18) at run
// granularity before the local UF:
//  L2 every run takes as parent the leftmost run of the row above it touches
//     (atomicMin of upper run starts: lower indices, so P[l] <= l throughout);
//  L3 row-column unification: every run walks its parent chain to its end and
//     records it (chains bounded by TY);
//  L4 local UF (Alg. 1 l.25-33) on the remaining adjacencies, most of which are
//     dismissed by one comparison of the coarse labels.
// Without COARSE_COLUMN, L4 runs directly on the run adjacencies (measured
// faster on B200).  L5 flattens: every run start
// points at its local root.
template <int TY, int CONN, bool COARSE_COLUMN = false>
__device__ __forceinline__ void tile_local_uf(TileSmem<TY>& sm, int warp, int lane) {
    __syncthreads();
    volatile int32_t* V = sm.P;
    if (COARSE_COLUMN) {
        for (int r = warp + 1; r < TY; r += kWarps)
            for_each_row_event<TY, CONN>(sm, r, lane, [&](int cs, int us) { atomicMin(&sm.P[cs >> 1], us); });
        __syncthreads();
        for (int r = warp + 1; r < TY; r += kWarps)
            for_each_run_start<TY>(sm, r, lane, [&](int l) {
                int t = l, p = V[l >> 1];
                while (p != t) {
                    t = p;
                    p = V[t >> 1];
                    V[l >> 1] = t;
                }
            });
        __syncthreads();
        for (int r = warp + 1; r < TY; r += kWarps)
            for_each_row_event<TY, CONN>(sm, r, lane, [&](int cs, int us) {
                if (V[cs >> 1] != V[us >> 1]) union_s(sm.P, cs, us);
            });
    } else {
        for (int r = warp + 1; r < TY; r += kWarps)
            for_each_row_event<TY, CONN>(sm, r, lane, [&](int cs, int us) { union_s(sm.P, cs, us); });
    }
    __syncthreads();
    for (int r = warp; r < TY; r += kWarps)
        for_each_run_start<TY>(sm, r, lane, [&](int l) { V[l >> 1] = find_s_ro(sm.P, l); });
    __syncthreads();
}

// Edge enumeration shared by K1 (write G) and K3 (flag roots): calls f(l, ls)
// for every foreground tile-edge item, l = tile-local index of the edge pixel,
// ls = tile-local index of the run start owning it (P[ls>>1] is its root after
// flattening).  Items: top-row run starts (if a tile is above), bottom-row run
// starts (if a tile is below), left-column pixels (if a tile is left),
// right-column pixels (if a tile is right).  K1 and K3 enumerate the same set,
// so K3 reads G only where K1 wrote it.
template <int TY, typename F>
__device__ __forceinline__ void for_each_edge_item(const TileSmem<TY>& sm, const Geom& g,
                                                   const TileId& id, int warp, int lane, F f) {
    const int rows = min(TY, g.H - id.y0);
    if (warp == 0 && id.y0 > 0) {
        uint32_t t = sm.wd[0][lane].s;
        while (t) {
            const int bit = __ffs(t) - 1;
            t &= t - 1;
            const int l = (lane << 5) + bit;
            f(l, l);
        }
    } else if (warp == 1 && id.y0 + TY < g.H) {
        uint32_t t = sm.wd[TY - 1][lane].s;
        while (t) {
            const int bit = __ffs(t) - 1;
            t &= t - 1;
            const int l = (TY - 1) * kTileW + (lane << 5) + bit;
            f(l, l);
        }
    } else if (warp == 2 && id.x0 > 0) {
        for (int r = lane; r < rows; r += 32)
            if (sm.wd[r][0].m & 1u) f(r * kTileW, r * kTileW);
    } else if (warp == 3 && id.x0 + kTileW < g.W) {
        for (int r = lane; r < rows; r += 32)
            if (sm.wd[r][kWords - 1].m >> 31)
                f(r * kTileW + kTileW - 1, r * kTileW + run_start_x(sm.wd[r], kTileW - 1));
    }
}

// =========================================================== K1: local merge
template <int TY, int CONN, bool VEC>
__global__ void __launch_bounds__(kThreads) k_local_merge(const uint8_t* __restrict__ img, Geom g,
                                                          uint32_t* __restrict__ bits,
                                                          int32_t* __restrict__ G,
                                                          uint16_t* __restrict__ R) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem<TY>& sm = *reinterpret_cast<TileSmem<TY>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const TileId id = decode_tile<TY>(g, blockIdx.x);
    const uint8_t* im = img + size_t(id.b) * size_t(g.npx);
    uint32_t* bm = bits + size_t(id.b) * size_t(g.nwords);

    for (int i = threadIdx.x; i < TY * kTileW / 64; i += kThreads) sm.flag[i] = 0;
    // Alg. 1 l.3-8: load the tile (out-of-image pixels read as background, R5)
    for (int r = warp; r < TY; r += kWarps) {
        const int y = id.y0 + r;
        uint32_t m = 0;
        if (VEC) {
            uint32_t h0 = 0, h1 = 0;
            if (y < g.H) {
                const uint8_t* row = im + size_t(y) * size_t(g.W) + id.x0;
                if (id.x0 + 16 * lane < g.W) h0 = nz16(ld_stream_u4(row + 16 * lane));
                if (id.x0 + 512 + 16 * lane < g.W) h1 = nz16(ld_stream_u4(row + 512 + 16 * lane));
            }
            const int src = (2 * lane) & 31;
            const uint32_t a0 = __shfl_sync(kFull, h0, src), a1 = __shfl_sync(kFull, h0, src + 1);
            const uint32_t b0 = __shfl_sync(kFull, h1, src), b1 = __shfl_sync(kFull, h1, src + 1);
            m = lane < 16 ? (a0 | (a1 << 16)) : (b0 | (b1 << 16));
        } else {
            const uint8_t* row = im + size_t(y < g.H ? y : 0) * size_t(g.W);
#pragma unroll 4
            for (int k = 0; k < kWords; ++k) {
                const int x = id.x0 + (k << 5) + lane;
                const bool fg = (y < g.H && x < g.W) ? (row[x] != 0) : false;
                const uint32_t bal = __ballot_sync(kFull, fg);
                if (lane == k) m = bal;
            }
        }
        const int wg = id.tx * kWords + lane;
        if (y < g.H && wg < g.WW) bm[size_t(y) * g.WW + wg] = m;
        tile_row_init<TY, true>(sm, r, lane, m);
    }
    tile_local_uf<TY, CONN>(sm, warp, lane);

    // Alg. 1 l.34-39 for tile-edge items only: G[g(l)] = g(root), G[g(root)] = g(root);
    // and flag the roots whose component touches a tile edge
    int32_t* Gb = G + size_t(id.b) * size_t(g.npx);
    const int W = g.W, x0 = id.x0, y0 = id.y0;
    for_each_edge_item<TY>(sm, g, id, warp, lane, [&](int l, int ls) {
        const int root = sm.P[ls >> 1];
        const int gl = (y0 + (l >> 10)) * W + x0 + (l & 1023);
        const int gr = (y0 + (root >> 10)) * W + x0 + (root & 1023);
        Gb[gl] = gr;
        Gb[gr] = gr;
        atomicOr(&sm.flag[root >> 6], 1u << ((root >> 1) & 31));
    });
    __syncthreads();
    // per-run records for K3 (local root + edge flag), runs in raster order
    uint16_t* Rt = R + size_t(blockIdx.x) * runs_per_tile_cap<TY>();
    for (int r = warp; r < TY; r += kWarps) {
        const int k0 = row_run_base<TY>(sm, r, lane) + sm.wd[r][lane].pad;
        int j = 0;
        for_each_run_start<TY>(sm, r, lane, [&](int l) {
            const int root = sm.P[l >> 1];
            const int e = (sm.flag[root >> 6] >> ((root >> 1) & 31)) & 1u;
            Rt[k0 + j++] = uint16_t(root | (e ? kRunEdgeBit : 0));
        });
    }
}

// ============================================================ K2: boundary
// Warp-cooperative union of a batch of (run start / edge pixel) index pairs:
// each lane holds at most one pair (ia, ib) (ia < 0: none).  Step 1 reads the
// local roots G[ia], G[ib] written by K1 (one independent load per lane);
// step 2 drops pairs already seen in this warp (identical root pairs are
// common: two large components meet at many places along a tile edge) so only
// one lane per distinct pair runs the global min-union.  This keeps the hot
// root of a giant component from being read once per crossing edge.
__device__ __forceinline__ void warp_union_pairs(int32_t* G, int ia, int ib, unsigned long long& last,
                                                 int img) {
    int a = -1, b = -1;
    if (ia >= 0) {
        a = ld_volatile(G + ia);
        b = ld_volatile(G + ib);
        if (a > b) { int t = a; a = b; b = t; }
    }
    const unsigned long long key =
        (ia >= 0 && a != b) ? ((unsigned long long)(unsigned)a << 32) | (unsigned)b : ~0ull;
    // pairs are only equal within one image (G values are image-local indices)
    const unsigned grp = __match_any_sync(kFull, key) & __match_any_sync(kFull, img);
    const int lane = threadIdx.x & 31;
    if (key != ~0ull && key != last && (__ffs(grp) - 1) == lane) union_g(G, a, b);
    if (key != ~0ull) last = key;
}

// Horizontal tile edges: one warp per (image, band >= 1, tile column); vertical
// tile edges: one thread per (image, tile column boundary >= 1, row).
template <int TY, int CONN>
__global__ void __launch_bounds__(256) k_boundary(Geom g, const uint32_t* __restrict__ bits,
                                                  int32_t* __restrict__ G, long long n_h,
                                                  long long blocks_h) {
    __shared__ Word s_w[8][2][kWords];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long last = ~0ull;
    if (blockIdx.x < blocks_h) {
        const long long task = (long long)blockIdx.x * 8 + warp;
        if (task >= n_h) return;  // whole warp exits together
        long long t = task;
        const int tx = int(t % g.tiles_x);
        t /= g.tiles_x;
        const int band = 1 + int(t % (g.tiles_y - 1));
        const int b = int(t / (g.tiles_y - 1));
        const int x0 = tx * kTileW, y0 = band * TY;
        const uint32_t* bm = bits + size_t(b) * size_t(g.nwords);
        int32_t* Gb = G + size_t(b) * size_t(g.npx);
        const int wg = tx * kWords + lane;
        const uint32_t cur = wg < g.WW ? bm[size_t(y0) * g.WW + wg] : 0u;
        const uint32_t up = wg < g.WW ? bm[size_t(y0 - 1) * g.WW + wg] : 0u;
        uint32_t sc, su;
        int cc, cu;
        row_runs(cur, lane, sc, cc);
        row_runs(up, lane, su, cu);
        s_w[warp][0][lane] = Word{cur, sc, cc, 0};
        s_w[warp][1][lane] = Word{up, su, cu, 0};
        __syncwarp();
        uint32_t curL = __shfl_up_sync(kFull, cur, 1), upL = __shfl_up_sync(kFull, up, 1);
        uint32_t curR = __shfl_down_sync(kFull, cur, 1), upR = __shfl_down_sync(kFull, up, 1);
        if (lane == 0) { curL = 0; upL = 0; }
        if (lane == 31) { curR = 0; upR = 0; }
        const uint32_t o = cur & up, oL = curL & upL;
        uint32_t ev = o & ~((o << 1) | (oL >> 31));
        uint32_t ne = 0, nw = 0;
        bool cnw = false, cne = false;  // diagonal edges through the tile corners
        if (CONN == 8) {
            const uint32_t cur_n = (cur >> 1) | (curR << 31), up_n = (up >> 1) | (upR << 31);
            const uint32_t cur_p = (cur << 1) | (curL >> 31), up_p = (up << 1) | (upL >> 31);
            ne = cur & ~cur_n & ~up & up_n;
            nw = cur & ~cur_p & ~up & up_p;
            if (lane == 0 && tx > 0 && (cur & 1u)) cnw = bm[size_t(y0 - 1) * g.WW + wg - 1] >> 31;
            if (lane == 31 && x0 + kTileW < g.W && (cur >> 31)) cne = bm[size_t(y0 - 1) * g.WW + wg + 1] & 1u;
        }
        const int gc = y0 * g.W + x0, gu = (y0 - 1) * g.W + x0, xb = lane << 5;
        while (__any_sync(kFull, ev | ne | nw | cnw | cne)) {
            int ia = -1, ib = -1;
            if (ev) {
                const int x = xb + __ffs(ev) - 1;
                ev &= ev - 1;
                ia = gc + run_start_x(s_w[warp][0], x);
                ib = gu + run_start_x(s_w[warp][1], x);
            } else if (ne) {
                const int x = xb + __ffs(ne) - 1;
                ne &= ne - 1;
                ia = gc + run_start_x(s_w[warp][0], x);
                ib = gu + x + 1;
            } else if (nw) {
                const int x = xb + __ffs(nw) - 1;
                nw &= nw - 1;
                ia = gc + x;
                ib = gu + run_start_x(s_w[warp][1], x - 1);
            } else if (cnw) {
                cnw = false;
                ia = gc;            // (x0, y0)
                ib = gu - 1;        // (x0-1, y0-1)
            } else if (cne) {
                cne = false;
                ia = gc + kTileW - 1;  // (x0+1023, y0)
                ib = gu + kTileW;      // (x0+1024, y0-1)
            }
            warp_union_pairs(Gb, ia, ib, last, 0);
        }
    } else {
        const long long task = (long long)(blockIdx.x - blocks_h) * 256 + threadIdx.x;
        const int nbx = g.tiles_x - 1;
        const long long n_v = (long long)g.B * g.H * nbx;
        const bool valid = task < n_v;
        long long t = valid ? task : 0;
        const int y = int(t % g.H);
        t /= g.H;
        const int bx = 1 + int(t % nbx);
        const int b = int(t / nbx);
        const int x0 = bx * kTileW;
        const uint32_t* bm = bits + size_t(b) * size_t(g.nwords);
        int32_t* Gb = G + size_t(b) * size_t(g.npx);
        const int wl = bx * kWords - 1;
        const size_t row = size_t(y) * g.WW;
        bool L = false, R = false, Lu = false, Ru = false;
        if (valid) {
            L = bm[row + wl] >> 31;
            R = bm[row + wl + 1] & 1u;
            if (CONN == 8 && (y % TY) != 0 && (L || R)) {
                Lu = bm[row - g.WW + wl] >> 31;
                Ru = bm[row - g.WW + wl + 1] & 1u;
            }
        }
        const int p = y * g.W + x0;
        warp_union_pairs(Gb, (L && R) ? p - 1 : -1, p, last, b);              // W edge of (x0, y)
        if (CONN == 8) {
            warp_union_pairs(Gb, (R && Lu) ? p : -1, p - g.W - 1, last, b);   // NW of (x0, y)
            warp_union_pairs(Gb, (L && Ru) ? p - 1 : -1, p - g.W, last, b);   // NE of (x0-1, y)
        }
    }
}

// ================================================================ K3: link
// Final link (§2.3): the tile's runs are re-derived from the bit mask (run
// starts only, no union-find) and take their local root from K1's per-run
// records; roots whose component touches a tile edge are resolved through G
// (find); then every pixel gets 1 + its global root, or 0.
template <int TY, int CONN, bool VEC>
__global__ void __launch_bounds__(kThreads) k_link(Geom g, const uint32_t* __restrict__ bits,
                                                   int32_t* __restrict__ G,
                                                   const uint16_t* __restrict__ R,
                                                   int32_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem<TY>& sm = *reinterpret_cast<TileSmem<TY>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const TileId id = decode_tile<TY>(g, blockIdx.x);
    const uint32_t* bm = bits + size_t(id.b) * size_t(g.nwords);
    int32_t* Gb = G + size_t(id.b) * size_t(g.npx);
    int32_t* ob = out + size_t(id.b) * size_t(g.npx);
    const uint16_t* Rt = R + size_t(blockIdx.x) * runs_per_tile_cap<TY>();

    for (int r = warp; r < TY; r += kWarps) {
        const int y = id.y0 + r;
        const int wg = id.tx * kWords + lane;
        const uint32_t m = (y < g.H && wg < g.WW) ? __ldg(bm + size_t(y) * g.WW + wg) : 0u;
        tile_row_init<TY, false>(sm, r, lane, m);
    }
    __syncthreads();

    // pass A: P[l] <- local root (untagged) for non-roots; roots get their
    // tagged final label 1 + global root
    const int W = g.W, x0 = id.x0, y0 = id.y0;
    for (int r = warp; r < TY; r += kWarps) {
        const int k0 = row_run_base<TY>(sm, r, lane) + sm.wd[r][lane].pad;
        int j = 0;
        for_each_run_start<TY>(sm, r, lane, [&](int l) {
            const int v = __ldg(Rt + k0 + j++);
            const int root = v & (kRunEdgeBit - 1);
            if (root == l) {
                int gr = (y0 + r) * W + x0 + (l & 1023);
                if (v & kRunEdgeBit) gr = find_g(Gb, gr);
                sm.P[l >> 1] = (gr + 1) | kTag;
            } else {
                sm.P[l >> 1] = root;
            }
        });
    }
    __syncthreads();
    // pass B: non-root run starts take their root's tagged label
    for (int r = warp; r < TY; r += kWarps)
        for_each_run_start<TY>(sm, r, lane, [&](int l) {
            const int p = sm.P[l >> 1];
            if (p >= 0) sm.P[l >> 1] = sm.P[p >> 1];
        });
    __syncthreads();

    // stream the labels; every run-start entry of P now holds its tagged label
    for (int r = warp; r < TY; r += kWarps) {
        const int y = y0 + r;
        if (y >= g.H) break;
        int32_t* orow = ob + size_t(y) * size_t(W) + x0;
        const int rb = r * kTileW;
        if (VEC) {
            // lane writes 4 consecutive pixels per step (512 B per warp store)
#pragma unroll 2
            for (int j = 0; j < kTileW / 128; ++j) {
                const int x = 128 * j + 4 * lane;
                if (x0 + x >= W) break;
                const int w = x >> 5, sh = x & 31;
                const Word wd = sm.wd[r][w];
                const uint32_t fgn = (wd.m >> sh) & 0xFu;
                int v0 = 0, v1 = 0, v2 = 0, v3 = 0;
                if (fgn) {
                    const uint32_t stn = (wd.s >> sh) & 0xFu;
                    int cur = 0;
                    if (fgn & 1u) {
                        const uint32_t below = wd.s & (kFull >> (31 - sh));
                        const int st = below ? ((w << 5) + 31 - __clz(below)) : wd.c;
                        cur = sm.P[(rb + st) >> 1];
                    }
                    const int pb = (rb + x) >> 1;  // P index of pixel x+1 / x+2 / x+3 starts
                    v0 = cur;
                    if (stn & 2u) cur = sm.P[pb];          // start at x+1: (rb+x+1)>>1 == pb
                    v1 = cur;
                    if (stn & 4u) cur = sm.P[pb + 1];      // start at x+2
                    v2 = cur;
                    if (stn & 8u) cur = sm.P[pb + 1];      // start at x+3: (rb+x+3)>>1 == pb+1
                    v3 = cur;
                    v0 = (fgn & 1u) ? (v0 & 0x7FFFFFFF) : 0;
                    v1 = (fgn & 2u) ? (v1 & 0x7FFFFFFF) : 0;
                    v2 = (fgn & 4u) ? (v2 & 0x7FFFFFFF) : 0;
                    v3 = (fgn & 8u) ? (v3 & 0x7FFFFFFF) : 0;
                }
                st_stream_i4(orow + x, v0, v1, v2, v3);
            }
        } else {
            for (int k = 0; k < kWords; ++k) {
                const int x = (k << 5) + lane;
                if (x0 + x < W) {
                    const uint32_t m = sm.wd[r][k].m;
                    int v = 0;
                    if ((m >> lane) & 1u) {
                        const int st = run_start_x(sm.wd[r], x);
                        v = sm.P[(rb + st) >> 1] & 0x7FFFFFFF;
                    }
                    orow[x] = v;
                }
            }
        }
    }
}

}  // namespace ccl
