// ccl_strip.cuh -- row-strip sharding of one gigapixel image over k GPUs
// (BASELINE.json north_star: "a single gigapixel image splits into row strips
// whose edge-row labels are exchanged with NCCL over NVLink, then merged by a
// cross-strip boundary-union and relabel pass").
//
// Per rank r (strip = rows [row0, row0 + rows) of the H_total x W image):
//   ccl_strip_local    K1 + K2 on the strip, with the strip's first / last rows
//                      treated as tile edges and labels offset by row0*W so they
//                      are global raster indices; then the strip's top and
//                      bottom rows' labels (2W) and, for each of those 2W slots,
//                      the first slot of the same row pair carrying the same
//                      label (2W "reps") -> the 4W-int send buffer.
//   (caller)           all-gather of the k send buffers (NCCL over NVLink).
//   ccl_strip_finalize min-union over the k*2W slots (same-label reps within a
//                      strip, and the 4-/8-adjacencies across every strip cut),
//                      minimum label per slot set, patch the strip's resolved
//                      edge labels F, then K3 writes the strip's labels.
// The union of canonical strip labelings is the canonical full labeling: a
// component's label is the minimum over its strip pieces' labels, since each
// piece's label is 1 + the minimum raster index of that piece.
#pragma once
#include "ccl_kernels.cuh"

namespace ccl {

// K2 tail in strip mode: as k_resolve, and marks Gs[root] = -1 for every edge
// root ("not on a strip boundary row" until k_strip_edges says otherwise).
// Gs is strip-local scratch (the labels_out buffer, overwritten by K3 later).
template <int TY>
__global__ void __launch_bounds__(256) k_strip_mark(Geom g, const int32_t* __restrict__ E,
                                                    const int32_t* __restrict__ F, int32_t* __restrict__ Gs,
                                                    unsigned ntiles) {
    const int lane = threadIdx.x & 31;
    for (unsigned t = (blockIdx.x * 256u + threadIdx.x) >> 5; t < ntiles; t += (gridDim.x * 256u) >> 5) {
        const int n = E[size_t(t) * kEdgeCap];
        for (int i = lane; i < n; i += 32) Gs[F[edge_slot(g.ntiles, i, t)] - 1 - g.label_off] = -1;
    }
}

// Labels of the strip's first (which = 0) and last (which = 1) image rows, one
// warp per (tile column, which); also Gs[root] = INT_MAX for their roots.
template <int TY>
__global__ void __launch_bounds__(256) k_strip_edges(Geom g, const uint32_t* __restrict__ bits,
                                                     const uint32_t* __restrict__ R,
                                                     const int32_t* __restrict__ E,
                                                     const int32_t* __restrict__ F,
                                                     int32_t* __restrict__ send, int32_t* __restrict__ Gs) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int task = blockIdx.x * 8 + warp;
    if (task >= 2 * g.tiles_x) return;
    const int tx = task >> 1, which = task & 1;
    const int y = which ? g.H - 1 : 0;
    const int band = y / TY;
    const size_t t = size_t(band) * g.tiles_x + tx;
    const int rbase = which ? E[t * kEdgeCap + 1] : 0;  // first run id of the band's last valid row
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
    const uint32_t* Rt = R + t * runs_per_tile_cap<TY>();
    const int x0 = tx * kTileW;
    for (int bit = 0; bit < 32; ++bit) {
        const int x = x0 + (lane << 5) + bit;
        if (x >= g.W) break;
        int lab = 0;
        if ((m >> bit) & 1u) {
            const int idx = pad + __popc(s & (kFull >> (31 - bit))) - 1;
            const uint32_t rec = Rt[rbase + idx];
            const int e = int(rec >> 16), rr = int(rec & 0x7FFFu);
            lab = e ? F[edge_slot(g.ntiles, e - 1, unsigned(t))] : (band * TY + (rr >> 10)) * g.W + x0 + (rr & 1023) + 1 + g.label_off;
            Gs[lab - 1 - g.label_off] = INT_MAX;
        }
        send[which * g.W + x] = lab;
    }
}

// Gs[root] = min slot index carrying that root's label (after k_strip_edges).
__global__ void k_strip_min(const int32_t* __restrict__ send, int32_t* __restrict__ Gs, int W, int label_off) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < 2 * W; s += gridDim.x * blockDim.x) {
        const int lab = send[s];
        if (lab) atomicMin(&Gs[lab - 1 - label_off], s);
    }
}

// rep[s] = first slot with the same label (into the send buffer's second half).
__global__ void k_strip_rep(int32_t* __restrict__ send, const int32_t* __restrict__ Gs, int W, int label_off) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < 2 * W; s += gridDim.x * blockDim.x) {
        const int lab = send[s];
        send[2 * W + s] = lab ? Gs[lab - 1 - label_off] : -1;
    }
}

// ---------------------------------------------------------------- finalize
// gathered: k blocks of 4W ints (rank order): top labels, bottom labels, reps.
// Slot id s = i*2W + j (strip i, j < W: top row x = j; j >= W: bottom row x = j - W).
__global__ void k_slots_init(int32_t* __restrict__ P, int32_t* __restrict__ minlab, int n) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
        P[s] = s;
        minlab[s] = INT_MAX;
    }
}

template <int CONN>
__global__ void k_slots_union(const int32_t* __restrict__ gathered, int32_t* __restrict__ P, int k, int W) {
    const int n = k * 2 * W;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
        const int i = s / (2 * W), j = s - i * 2 * W;
        const int32_t* blk = gathered + size_t(i) * 4 * W;
        if (!blk[j]) continue;
        const int rep = blk[2 * W + j];
        if (rep != j) union_g(P, s, i * 2 * W + rep);  // same piece within strip i
        if (j >= W && i + 1 < k) {                       // bottom row of strip i vs top row of i+1
            const int x = j - W;
            const int32_t* nxt = gathered + size_t(i + 1) * 4 * W;
            for (int dx = (CONN == 8 ? -1 : 0); dx <= (CONN == 8 ? 1 : 0); ++dx) {
                const int xx = x + dx;
                if (xx >= 0 && xx < W && nxt[xx]) union_g(P, s, (i + 1) * 2 * W + xx);
            }
        }
    }
}

__global__ void k_slots_minlab(const int32_t* __restrict__ gathered, const int32_t* __restrict__ P,
                               int32_t* __restrict__ minlab, int k, int W) {
    const int n = k * 2 * W;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
        const int i = s / (2 * W), j = s - i * 2 * W;
        const int lab = gathered[size_t(i) * 4 * W + j];
        if (lab) atomicMin(&minlab[find_g_ro(P, s)], lab);
    }
}

// Patch this rank's resolved edge labels F for components on its boundary rows.
template <int TY>
__global__ void __launch_bounds__(256) k_strip_patch(Geom g, const int32_t* __restrict__ E, int32_t* __restrict__ F,
                                                     const int32_t* __restrict__ Gs, const int32_t* __restrict__ P,
                                                     const int32_t* __restrict__ minlab, int rank, unsigned ntiles) {
    const int lane = threadIdx.x & 31;
    const int slot0 = rank * 2 * g.W;
    for (unsigned t = (blockIdx.x * 256u + threadIdx.x) >> 5; t < ntiles; t += (gridDim.x * 256u) >> 5) {
        const int n = E[size_t(t) * kEdgeCap];
        for (int i = lane; i < n; i += 32) {
            int32_t* f = F + edge_slot(g.ntiles, i, t);
            const int v = Gs[*f - 1 - g.label_off];
            if (v >= 0) *f = minlab[find_g_ro(P, slot0 + v)];
        }
    }
}

}  // namespace ccl
