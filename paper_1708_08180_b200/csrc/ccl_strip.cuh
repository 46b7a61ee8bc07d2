// ccl_strip.cuh -- row-strip sharding of one gigapixel image over k GPUs
// (BASELINE.json north_star: "a single gigapixel image splits into row strips
// whose edge-row labels are exchanged with NCCL over NVLink, then merged by a
// cross-strip boundary-union and relabel pass").  The
// decomposition is the paper's tile decomposition (§2.1.1) and
// boundary merge (§2.2) one level up: a strip is labeled alone,
// then only the cells on the strip boundaries are merged.
//
// Per rank r (strip = rows [row0, row0 + rows) of the H_total x W image), six
// launches per step plus the collective:
//   ccl_strip_local    K1 (the strip's first / last rows count as tile edges;
//                      every edge slot's strip mark F[slot] = -1), K2,
//                      k_strip_edges (labels of the strip's top and bottom
//                      rows: each boundary run's edge root resolved in G; per
//                      root the first boundary slot carrying it, by atomicMax
//                      of INT_MAX - slot into F[root]),
//                      k_strip_rep (the 4W-int send buffer's second half: for
//                      each boundary slot, the first slot with the same root;
//                      and the slot union-find initialised)
//   (caller)           all-gather of the k send buffers (NCCL over NVLink)
//   ccl_strip_finalize k_slots_union (min-label union over the k*2W slots:
//                      same-root slots of a strip, and the 4-/8-adjacencies
//                      across every strip cut), K3 (its helper warp resolves
//                      each edge root in G and, for roots on a strip boundary,
//                      takes the minimum label of their slot set).
// The union of canonical strip labelings is the canonical full labeling: a
// component's label is the minimum over its strip pieces' labels, since each
// piece's label is 1 + the minimum raster index of that piece.
#pragma once
#include <climits>

#include "ccl_kernels.cuh"

namespace ccl {

// Slot union-find of the finalize step: P[s] = ~0 (a root) or the key of s's
// parent, key(s) = (label of s << 32) | s.  A set's root is its slot with the
// smallest label (ties: smallest slot), so the root key's high word is the
// set's minimum label -- no separate minimum pass.
constexpr uint64_t kSlotRoot = ~0ull;

__device__ __forceinline__ uint64_t slot_key(const int32_t* gathered, int W, unsigned s) {
    const unsigned i = s / unsigned(2 * W), j = s - i * unsigned(2 * W);
    return (uint64_t(uint32_t(gathered[size_t(i) * 4 * W + j])) << 32) | s;
}

// root key of slot s (path halving: s re-pointed at its grandparent)
__device__ __forceinline__ uint64_t slot_find(uint64_t* P, const int32_t* gathered, int W, unsigned s) {
    uint64_t v = __ldcg(reinterpret_cast<const unsigned long long*>(P) + s);
    if (v == kSlotRoot) return slot_key(gathered, W, s);
    CCL_LOOP_GUARD(sf);
    while (true) {
        CCL_LOOP_TICK(sf);
        const unsigned p = unsigned(v);
        const uint64_t w = __ldcg(reinterpret_cast<const unsigned long long*>(P) + p);
        if (w == kSlotRoot) return v;  // p is the root: v is its key
        __stcg(reinterpret_cast<unsigned long long*>(P) + s, static_cast<unsigned long long>(w));
        s = p;
        v = w;
    }
}

__device__ __forceinline__ void slot_union(uint64_t* P, const int32_t* gathered, int W, unsigned a, unsigned b) {
    CCL_LOOP_GUARD(su);
    while (true) {
        CCL_LOOP_TICK(su);
        uint64_t ka = slot_find(P, gathered, W, a), kb = slot_find(P, gathered, W, b);
        if (ka == kb) return;
        if (ka < kb) { const uint64_t t = ka; ka = kb; kb = t; }
        const uint64_t old = atomicMin(reinterpret_cast<unsigned long long*>(P) + unsigned(ka),
                                       static_cast<unsigned long long>(kb));
        if (old == kSlotRoot) return;  // ka's slot was a root: linked under kb
        a = unsigned(old);             // re-linked meanwhile: union what was displaced
        b = unsigned(kb);
    }
}

// Labels of the strip's first (which = 0) and last (which = 1) image rows, one
// warp per (tile column, which).  For each boundary pixel: its edge root
// (resolved in G) gives the label; each run's first pixel posts its slot to
// F[root] (atomicMax of INT_MAX - slot: the first boundary slot of the root);
// send[2W + slot] = the root's slot for k_strip_rep (-1: background, -2: a
// run of the image's own first / last row whose component touches no edge).
template <int TY>
__global__ void __launch_bounds__(256) k_strip_edges(Geom g, const uint32_t* __restrict__ bits,
                                                     const uint32_t* __restrict__ R,
                                                     const int32_t* __restrict__ E, uint64_t* __restrict__ G,
                                                     int32_t* __restrict__ F, int32_t* __restrict__ send) {
    pdl_wait();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int task = blockIdx.x * 8 + warp;
    if (task >= 2 * g.tiles_x) return;
    const int tx = task >> 1, which = task & 1;
    const int y = which ? g.H - 1 : 0;
    const int band = y / TY;
    const unsigned t = unsigned(band) * unsigned(g.tiles_x) + unsigned(tx);
    const int rbase = which ? E[size_t(t) * kEdgeCap + 1] : 0;  // first run id of the band's last valid row
    const int wg = tx * kWords + lane;
    const uint32_t m = wg < g.WW ? bits[size_t(y) * g.WW + wg] : 0u;
    uint32_t pm = __shfl_up_sync(kFull, m, 1);
    if (lane == 0) pm = 0;
    const uint32_t s = m & ~((m << 1) | (pm >> 31));
    int incl = __popc(s);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += u;
    }
    const int pad = incl - __popc(s);
    const uint32_t* Rt = R + size_t(t) * runs_per_tile_cap<TY>();
    const int x0 = tx * kTileW;
    int lab = 0, root = -1, cur_idx = -1;
    for (int bit = 0; bit < 32; ++bit) {
        const int x = x0 + (lane << 5) + bit;
        if (x >= g.W) break;
        const int slot = which * g.W + x;
        if ((m >> bit) & 1u) {
            const int idx = pad + __popc(s & (kFull >> (31 - bit))) - 1;
            if (idx != cur_idx) {  // a new run (or the run entering this word): resolve its root once
                cur_idx = idx;
                const uint32_t rec = Rt[rbase + idx];
                if (rec >> 16) {
                    const uint64_t w = resolve_slot(G, edge_slot(g.ntiles, int(rec >> 16) - 1, t));
                    root = int(unsigned(w));
                    lab = int(w >> 32) + 1 + g.label_off;
                } else {  // the image's own top / bottom row (first / last strip): not an edge root
                    const int rr = int(rec & 0x7FFFu);
                    root = -2;
                    lab = (band * TY + (rr >> 10)) * g.W + x0 + (rr & 1023) + 1 + g.label_off;
                }
            }
            if (root >= 0 && ((s >> bit) & 1u || bit == 0)) atomicMax(F + root, INT_MAX - slot);
            send[slot] = lab;
            send[2 * g.W + slot] = root;
        } else {
            send[slot] = 0;
            send[2 * g.W + slot] = -1;
        }
    }
}

// send[2W + s] = first slot with the same root (-1: background); and the
// slot union-find of the finalize step set to k * 2W roots.
__global__ void k_strip_rep(int32_t* __restrict__ send, const int32_t* __restrict__ F, uint64_t* __restrict__ P,
                            int W, int n_slots) {
    pdl_wait();
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < 2 * W; s += gridDim.x * blockDim.x) {
        const int root = send[2 * W + s];  // edge-root slot, -1 background, -2 no edge root (its own rep)
        send[2 * W + s] = root >= 0 ? INT_MAX - F[root] : (root == -2 ? s : -1);
    }
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_slots; s += gridDim.x * blockDim.x) P[s] = kSlotRoot;
}

// ---------------------------------------------------------------- finalize
// gathered: k blocks of 4W ints (rank order): top labels, bottom labels, reps.
// Slot id s = i*2W + j (strip i, j < W: top row x = j; j >= W: bottom row x = j - W).
template <int CONN>
__global__ void k_slots_union(const int32_t* __restrict__ gathered, uint64_t* __restrict__ P, int k, int W) {
    const int n = k * 2 * W;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
        const int i = s / (2 * W), j = s - i * 2 * W;
        const int32_t* blk = gathered + size_t(i) * 4 * W;
        if (!blk[j]) continue;
        const int rep = blk[2 * W + j];
        if (rep != j) slot_union(P, gathered, W, unsigned(s), unsigned(i * 2 * W + rep));  // one piece of strip i
        if (j >= W && i + 1 < k) {  // bottom row of strip i vs top row of strip i+1
            const int x = j - W;
            const int32_t* nxt = gathered + size_t(i + 1) * 4 * W;
            for (int dx = (CONN == 8 ? -1 : 0); dx <= (CONN == 8 ? 1 : 0); ++dx) {
                const int xx = x + dx;
                if (xx >= 0 && xx < W && nxt[xx]) slot_union(P, gathered, W, unsigned(s), unsigned((i + 1) * 2 * W + xx));
            }
        }
    }
}

}  // namespace ccl
