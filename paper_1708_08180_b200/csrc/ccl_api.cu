// ccl_api.cu -- host side of libccl.so: argument validation, launch geometry,
// workspace layout and the C ABI declared in include/ccl.h.
#include "../../include/ccl.h"
#include "ccl_kernels.cuh"
#include "ccl_strip.cuh"
#include "ccl_baselines.cuh"
#include "ccl_stats.cuh"
#include "ccl_3d.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <mutex>
#include <atomic>
#include <chrono>
#include <random>

namespace {

thread_local int g_last_cuda_error = 0;

constexpr int64_t kSmallTilesPerSM = 4;  // default tile height: the tallest giving this many tiles per SM
constexpr size_t kAlign = 256;

size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// A value unique to this call (per process; 64-bit, randomly seeded): the
// K1 -> K2 ready flags carry it, so flags left in a reused workspace by an
// earlier call never read as ready.
unsigned long long next_epoch() {
    static std::atomic<unsigned long long> counter{
        (std::random_device{}() * 0x9E3779B97F4A7C15ull) ^ (unsigned long long)std::chrono::steady_clock::now().time_since_epoch().count()};
    unsigned long long e;
    do { e = counter.fetch_add(0x9E3779B97F4A7C15ull) + 0x9E3779B97F4A7C15ull; } while (e == 0);
    return e;
}

// SMs of the current device (launch sizing)
int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 1;
    }
    return cached[dev];
}

struct Plan {
    ccl::Geom g;
    int ty;
    size_t G_bytes, bits_bytes, runs_bytes, edge_bytes, F_bytes, defer_bytes, ready_bytes;
    size_t strip_F_bytes;  // F (strip marks / resolved labels): strip stages only, else F_bytes = 0
    size_t total() const {
        return G_bytes + bits_bytes + runs_bytes + edge_bytes + F_bytes + defer_bytes + ready_bytes;
    }
};

ccl_status_t check_geometry(int64_t B, int64_t H, int64_t W, int conn) {
    if (B < 0 || H < 1 || W < 1) return CCL_ERR_DIMS;
    if (H > INT32_MAX / W) return CCL_ERR_TOO_LARGE;
    if (conn != 4 && conn != 8) return CCL_ERR_CONNECTIVITY;
    return CCL_OK;
}

ccl_status_t make_plan(int64_t B, int64_t H, int64_t W, int conn, int tile_rows, Plan& p) {
    ccl_status_t st = check_geometry(B, H, W, conn);
    if (st != CCL_OK) return st;
    if (tile_rows == 0) {
        // Default tile height: the tallest of 32 / 16 / 8 rows that still gives
        // the persistent K1 grid (SMs x 4-5 blocks) at least kSmallTilesPerSM
        // tiles per SM.  Taller tiles halve the boundaries K2 unions and the
        // tiles K3 walks (C3 8192^2 texture 113 -> 102.5 us at 32 rows); small
        // images are latency-bound per tile (C1 512^2 noise 74 -> 56 us and C2
        // 2048^2 noise 130 -> 102 us at 8 rows).  CCL_TILE_AUTO=0 pins it to 16.
        static const bool autoty = [] {
            const char* v = std::getenv("CCL_TILE_AUTO");
            return !(v && v[0] == '0');
        }();
        const int64_t tx = (W + ccl::kTileW - 1) / ccl::kTileW, need = kSmallTilesPerSM * sm_count();
        if (!autoty) tile_rows = 16;
        else if (B * tx * ((H + 31) / 32) >= need) tile_rows = 32;
        else if (B * tx * ((H + 15) / 16) >= need) tile_rows = 16;
        else tile_rows = 8;
    }
    if (tile_rows != 8 && tile_rows != 16 && tile_rows != 32) return CCL_ERR_CONFIG;
    if (B > INT32_MAX) return CCL_ERR_DIMS;
    p.ty = tile_rows;
    p.g.B = int(B);
    p.g.H = int(H);
    p.g.W = int(W);
    p.g.WW = int((W + 31) / 32);
    p.g.tiles_x = int((W + ccl::kTileW - 1) / ccl::kTileW);
    p.g.tiles_y = int((H + tile_rows - 1) / tile_rows);
    p.g.npx = H * W;
    p.g.nwords = H * int64_t(p.g.WW);
    p.g.div_tx = ccl::FastDiv(unsigned(p.g.tiles_x));
    p.g.div_ty = ccl::FastDiv(unsigned(p.g.tiles_y));
    p.g.div_ty1 = ccl::FastDiv(unsigned(std::max(1, p.g.tiles_y - 1)));
    p.g.div_tx1 = ccl::FastDiv(unsigned(std::max(1, p.g.tiles_x - 1)));
    p.g.div_vg = ccl::FastDiv(unsigned((p.g.tiles_y + 32 / tile_rows - 1) / (32 / tile_rows)));
    p.g.label_off = 0;
    p.g.force_top = 0;
    p.g.force_bottom = 0;
    p.g.k3_early = 1;
    p.g.strip = 0;
    p.g.epoch = 0;
    p.g.ready = nullptr;
    p.g.defer = nullptr;
    p.g.thr = 1;  // foreground = nonzero (ccl_label_threshold_async sets another threshold)
    p.g.thr_k = 0x7F7F7F7Fu;
    p.g.ntiles = unsigned(int64_t(B) * p.g.tiles_x * p.g.tiles_y);
    // edge slots (the boundary analysis' union-find nodes, 8 B each) and their
    // resolved labels in strip mode (4 B each): edge_slots(TY) per tile, sized
    // for the tile configuration that needs the most (ccl_kernels.cuh)
    const size_t tiles8 = size_t(B) * size_t(p.g.tiles_x) * size_t((H + 7) / 8);
    const size_t tiles16 = size_t(B) * size_t(p.g.tiles_x) * size_t((H + 15) / 16);
    const size_t tiles32 = size_t(B) * size_t(p.g.tiles_x) * size_t((H + 31) / 32);
    const size_t slots = std::max({tiles8 * ccl::edge_slots(8), tiles16 * ccl::edge_slots(16),
                                   tiles32 * ccl::edge_slots(32)});
    if (slots >= size_t(INT32_MAX)) return CCL_ERR_TOO_LARGE;
    p.G_bytes = align_up(slots * sizeof(uint64_t));
    p.strip_F_bytes = align_up(slots * sizeof(int32_t));
    p.F_bytes = 0;  // strip_plan / ccl_strip_workspace_bytes add it
    p.bits_bytes = align_up(size_t(B) * size_t(H) * size_t(p.g.WW) * sizeof(uint32_t));
    // per-run records: capacity of the worst case (alternating pixels) for the
    // tallest tile config, so the size does not depend on tile_rows
    const size_t rows32 = size_t((H + 31) / 32) * 32;
    p.runs_bytes = align_up(size_t(B) * size_t(p.g.tiles_x) * rows32 * (ccl::kTileW / 2) * sizeof(uint32_t));
    // edge briefs E: kEdgeCap ints per tile, for the most tiles any config
    // makes (tile_rows = 8)
    p.edge_bytes = align_up(tiles8 * ccl::kEdgeCap * sizeof(int32_t));
    p.ready_bytes = align_up(tiles8 * sizeof(uint64_t));  // per-tile ready flags (K1 -> K2 overlap)
    p.defer_bytes = align_up(tiles8 * sizeof(int32_t));   // K1's lists of run-dense tiles
    return CCL_OK;
}

ccl_status_t cuda_fail(cudaError_t e) {
    g_last_cuda_error = int(e);
    return CCL_ERR_CUDA;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
    const char* pa = static_cast<const char*>(a);
    const char* pb = static_cast<const char*>(b);
    return na && nb && pa < pb + nb && pb < pa + na;
}

template <int TY>
size_t smem_bytes() { return sizeof(ccl::LinkSmem<TY>); }

// the K3 kernel (TMA row stores / resolve in the helper warp)
template <int TY, int CONN, bool VEC, bool TMA, bool RES>
constexpr auto k3_kernel() {
    return ccl::k_link<TY, CONN, VEC, TMA, RES>;
}
template <int TY>
size_t smem_bytes_k1() { return sizeof(ccl::K1Smem<TY>); }

template <int TY, int CONN, bool VEC>
cudaError_t setup_attrs_now() {
#ifndef CCL_K2_CARVEOUT
#define CCL_K2_CARVEOUT 40
#endif
    // K2's finds are served from L1 (ld.global.ca): a 40 % shared-memory
    // carveout (100 KB: 5-6 resident 16 KB blocks) leaves the rest of the
    // 256 KB to L1.  Measured, C3 K2 µs: default (no hint) 26-29 and
    // varying between runs, 100 % 25, 40 % 24.5, 0 % 49 (blocks no
    // longer all resident); noise 80 / 65 / 56 / 149.
    cudaFuncSetAttribute(ccl::k_boundary<TY, CONN>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         CCL_K2_CARVEOUT);
    cudaError_t e = cudaFuncSetAttribute(ccl::k_local_merge<TY, CONN, VEC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem_bytes_k1<TY>()));
    if (e != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ccl::k_local_merge<TY, CONN, VEC, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem_bytes_k1<TY>()))) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(ccl::k_local_merge<TY, CONN, VEC, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem_bytes_k1<TY>()))) != cudaSuccess)
        return e;
    const int sm3 = int(smem_bytes<TY>());
    if ((e = cudaFuncSetAttribute(k3_kernel<TY, CONN, VEC, false, true>(),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, sm3)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(k3_kernel<TY, CONN, VEC, true, true>(),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, sm3)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(k3_kernel<TY, CONN, VEC, false, false>(),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, sm3)) != cudaSuccess)
        return e;
    return cudaFuncSetAttribute(k3_kernel<TY, CONN, VEC, true, false>(),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, sm3);
}

// Kernel attributes (> 48 KB dynamic shared memory opt-in, carveout) are
// per device: applied once per instantiation AND device (the current one).
template <int TY, int CONN, bool VEC>
cudaError_t setup_attrs() {
    constexpr int kMaxDev = 64;
    static std::mutex mu;
    static bool done[kMaxDev] = {false};
    static cudaError_t result[kMaxDev];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDev) return setup_attrs_now<TY, CONN, VEC>();
    std::lock_guard<std::mutex> lock(mu);
    if (!done[dev]) {
        result[dev] = setup_attrs_now<TY, CONN, VEC>();
        done[dev] = true;
    }
    return result[dev];
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// TMA descriptor of the int32 label tensor viewed as [B*H][W/32][32] with a
// [1][32][32] box (one 1024-px tile row) and 128-byte swizzle (W % 32 == 0).
bool encode_label_map(CUtensorMap* map, int32_t* out, const ccl::Geom& g) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {32, cuuint64_t(g.W / 32), cuuint64_t(g.B) * cuuint64_t(g.H)};
    const cuuint64_t strides[2] = {128, cuuint64_t(g.W) * 4};
    // box: a whole row (32 words x 32 px, SWIZZLE_128B) or, CCL_K3_SPLIT = 2 / 4,
    // a half / quarter of every word (32 words x 16 / 8 px, SWIZZLE_64B / 32B)
    const cuuint32_t box[3] = {cuuint32_t(32 / CCL_K3_SPLIT), 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUtensorMapSwizzle sw = CCL_K3_SPLIT == 4 ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : (CCL_K3_SPLIT == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Launch with programmatic stream serialisation (PDL): the kernel's blocks
// may be scheduled while the previous kernel on the stream drains; the kernel
// itself waits (griddepcontrol.wait) before touching its inputs.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool off = [] {
        const char* v = std::getenv("CCL_PDL");
        return v && v[0] == '0';
    }();
    cfg.attrs = attr;
    cfg.numAttrs = off ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

enum Stage { kK1 = 1, kK2 = 2, kK3 = 4, kAll = 7, kStripEdges = 8, kStripFinalize = 16 };

// Strip-mode arguments (row-strip sharding, ccl_strip_local / _finalize).
struct StripCtx {
    int32_t* send = nullptr;            // this rank's 4W send buffer
    const int32_t* gathered = nullptr;  // k * 4W, rank order
    int k = 1, rank = 0;
    uint64_t* P = nullptr;              // k * 2W slot union-find entries (ccl_strip.cuh)
};


// Resident blocks per device for the persistent kernels K1 (which = 1) and
// K3 (which = 3): SMs x blocks per SM at full occupancy, cached per
// instantiation and device.
template <int TY, int CONN, bool VEC>
int persistent_blocks(int which) {
    static int cached[2][64] = {{0}};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    const int w = which == 1 ? 0 : 1;
    if (cached[w][dev]) return cached[w][dev];
    int sms = 0, b = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (which == 1)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ccl::k_local_merge<TY, CONN, VEC>, ccl::k1_threads<TY>(),
                                                      smem_bytes_k1<TY>());
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k3_kernel<TY, CONN, VEC, true, true>(), ccl::kK3Threads,
                                                      smem_bytes<TY>());
    cached[w][dev] = std::max(1, sms) * std::max(1, b);
    return cached[w][dev];
}

template <int TY, int CONN, bool VEC>
cudaError_t run_stages(const Plan& p, int stages, const uint8_t* img, int32_t* out, void* ws,
                       cudaStream_t s, const StripCtx* sc) {
    cudaError_t e = setup_attrs<TY, CONN, VEC>();
    if (e != cudaSuccess) return e;
    ccl::Geom g = p.g;  // (per call: the K1 -> K2 overlap epoch below)
    uint64_t* G = static_cast<uint64_t*>(ws);
    uint32_t* bits = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + p.G_bytes);
    uint32_t* runs = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + p.G_bytes + p.bits_bytes);
    int32_t* E = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + p.G_bytes + p.bits_bytes + p.runs_bytes);
    int32_t* F = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(E) + p.edge_bytes);
    const long long ntiles = (long long)g.B * g.tiles_x * g.tiles_y;
    if (ntiles == 0) return cudaSuccess;
    const size_t smem = smem_bytes<TY>();
    // persistent K1/K3: one wave of resident blocks walks all tiles
    const unsigned grid1 = unsigned(std::min<long long>(ntiles, (long long)persistent_blocks<TY, CONN, VEC>(1)));
#ifdef CCL_K3_GRID  // timing experiments only (tools/build_variant.sh)
    const unsigned grid3 = unsigned(std::min<long long>(ntiles, (long long)CCL_K3_GRID));
#else
    const unsigned grid3 = unsigned(std::min<long long>(ntiles, (long long)persistent_blocks<TY, CONN, VEC>(3)));
#endif
    const long long n_h = (long long)g.B * (g.tiles_y - 1) * g.tiles_x;
    const long long n_v = (long long)g.B * ((g.tiles_y + ccl::v_bands<TY>() - 1) / ccl::v_bands<TY>()) *
                          (g.tiles_x - 1);
    g.epoch = 0;
    g.ready = nullptr;
    static const bool overlap = [] {
        const char* v = std::getenv("CCL_K1K2_OVERLAP");
        return !(v && v[0] == '0');
    }();
    if (overlap && (stages & kK1) && (stages & kK2) && n_h + n_v > 0) {
        g.epoch = next_epoch();
        g.ready = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + p.total() - p.ready_bytes);
    }
    g.defer = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + p.total() - p.ready_bytes - p.defer_bytes);
    if (stages & kK1) {
        // the foreground test: nonzero, or value >= thr (fused threshold, THR 1 / 2)
        auto k1 = g.thr == 1 ? ccl::k_local_merge<TY, CONN, VEC>
                             : (g.thr <= 128 ? ccl::k_local_merge<TY, CONN, VEC, 0, 1> : ccl::k_local_merge<TY, CONN, VEC, 0, 2>);
        k1<<<grid1, ccl::k1_threads<TY>(), smem_bytes_k1<TY>(), s>>>(img, g, bits, G, runs, E, F, unsigned(ntiles));
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (stages & kK2) {
        // K2: boundary unions (one warp per tile boundary), then resolve every
        // tile's edge-touching roots (one warp per tile)
        if (n_h + n_v > 0) {
            // few boundaries (small images): split each horizontal one over
            // 2 or 4 warps so the launch still fills the GPU (one task per
            // warp, ~5900 warps resident in one wave)
#ifndef CCL_K2_SUB_MIN
#define CCL_K2_SUB_MIN 0  // minimum split of a horizontal boundary: 2^SUB_MIN warps
#endif
            int sub_log2 = CCL_K2_SUB_MIN;
#ifndef CCL_K2_SUB_MAX
#define CCL_K2_SUB_MAX 2
#endif
            while (sub_log2 < CCL_K2_SUB_MAX && ((n_h << (sub_log2 + 1)) + n_v) <= (long long)sm_count() * 40)
                ++sub_log2;
#ifndef CCL_K2_DBG
#define CCL_K2_DBG 0  // timing experiments only (tools/build_variant.sh): 3 = skip K2, 4 = no unions
#endif
            e = launch_pdl(ccl::k_boundary<TY, CONN, CCL_K2_DBG>,
                           unsigned(((n_h << sub_log2) + n_v + ccl::kK2Warps - 1) / ccl::kK2Warps),
                           32 * ccl::kK2Warps, 0, s, g,
                           (const uint32_t*)bits, (const uint32_t*)runs, (const int32_t*)E, G, n_h, n_v, sub_log2);
            if (e != cudaSuccess) return e;
        }
        // the resolve step (edge roots -> final labels) runs in K3's helper warps
    }
    if (stages & kStripEdges) {
        // boundary-row labels + first slot per root (F), then the send
        // buffer's reps and the slot union-find's initial roots
        e = launch_pdl(ccl::k_strip_edges<TY>, unsigned((2 * g.tiles_x + 7) / 8), 256, 0, s, g,
                       (const uint32_t*)bits, (const uint32_t*)runs, (const int32_t*)E, G, F, sc->send);
        if (e != cudaSuccess) return e;
        const int n = sc->k * 2 * g.W;
        const unsigned sb = unsigned(std::min(sm_count() * 8, (n + 255) / 256));
        e = launch_pdl(ccl::k_strip_rep, sb, 256, 0, s, sc->send, (const int32_t*)F, sc->P, g.W, n);
        if (e != cudaSuccess) return e;
    }
    if (stages & kStripFinalize) {
        // after the caller's all-gather (a plain launch: it must not overlap it)
        const int n = sc->k * 2 * g.W;
        const unsigned sb = unsigned(std::min(sm_count() * 8, (n + 255) / 256));
        ccl::k_slots_union<CONN><<<sb, 256, 0, s>>>(sc->gathered, sc->P, sc->k, g.W);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (stages & kK3) {
        // K3 reads K1's outputs before its PDL wait unless K1 is its direct
        // predecessor in this call (an image with a single tile: no boundaries)
        ccl::Geom g3 = g;
        if ((stages & kK1) && !(stages & kStripFinalize)) {
            const long long nb = (long long)g.B * (g.tiles_y - 1) * g.tiles_x +
                                 (long long)g.B * ((g.tiles_y + ccl::v_bands<TY>() - 1) / ccl::v_bands<TY>()) *
                                     (g.tiles_x - 1);
            g3.k3_early = nb > 0;
        }
        // labels leave through TMA bulk-tensor stores when rows are 32-px
        // multiples (all bench configs); else 128-bit st.global.cs.  The
        // helper warp resolves the edge roots; in strip mode (!res) roots on
        // a strip boundary take their slot set's minimum label.
        CUtensorMap map;
        std::memset(&map, 0, sizeof(map));
        const bool tma = VEC && g.W % 32 == 0 && encode_label_map(&map, out, g);
        const bool res = !(stages & kStripFinalize);
        ccl::StripFinal sf{};
        if (!res) sf = ccl::StripFinal{F, sc->P, sc->gathered, g.W, sc->rank * 2 * g.W};
        auto k3 = tma ? (res ? k3_kernel<TY, CONN, VEC, true, true>() : k3_kernel<TY, CONN, VEC, true, false>())
                      : (res ? k3_kernel<TY, CONN, VEC, false, true>() : k3_kernel<TY, CONN, VEC, false, false>());
        e = launch_pdl(k3, grid3, ccl::kK3Threads, smem, s, g3, (const uint32_t*)bits, (const uint32_t*)runs,
                       (const int32_t*)E, G, sf, out, unsigned(ntiles), map);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <int TY>
cudaError_t dispatch_conn(const Plan& p, int conn, bool vec, int stages, const uint8_t* img,
                          int32_t* out, void* ws, cudaStream_t s, const StripCtx* sc) {
    if (conn == 4)
        return vec ? run_stages<TY, 4, true>(p, stages, img, out, ws, s, sc)
                   : run_stages<TY, 4, false>(p, stages, img, out, ws, s, sc);
    return vec ? run_stages<TY, 8, true>(p, stages, img, out, ws, s, sc)
               : run_stages<TY, 8, false>(p, stages, img, out, ws, s, sc);
}

// The 128-bit paths need 16-byte aligned rows: W % 16 == 0 for the uint8 image
// (which also gives W % 4 == 0 for the int32 labels) and aligned base pointers.
bool vector_ok(const Plan& p, const void* img, const void* out) {
    if (p.g.W % 16) return false;
    if (img && (reinterpret_cast<uintptr_t>(img) & 15)) return false;
    if (out && (reinterpret_cast<uintptr_t>(out) & 15)) return false;
    return true;
}

ccl_status_t run(const Plan& p, int conn, int stages, const uint8_t* img, int32_t* out, void* ws,
                 cudaStream_t s, const StripCtx* sc = nullptr) {
    const bool vec = vector_ok(p, img, out);
    cudaError_t e;
    switch (p.ty) {
        case 8: e = dispatch_conn<8>(p, conn, vec, stages, img, out, ws, s, sc); break;
        case 16: e = dispatch_conn<16>(p, conn, vec, stages, img, out, ws, s, sc); break;
        case 32: e = dispatch_conn<32>(p, conn, vec, stages, img, out, ws, s, sc); break;
        default: return CCL_ERR_CONFIG;
    }
    return e == cudaSuccess ? CCL_OK : cuda_fail(e);
}

template <int CONN>
cudaError_t run_method(int method, const uint8_t* img, int B, int H, int W, int32_t* out, void* ws, cudaStream_t s) {
    namespace cb = ccl::base;
    const long long npx = (long long)H * W, n = npx * B;
    const unsigned flat_blocks = unsigned(std::min<long long>((n + 255) / 256, (long long)sm_count() * 16));
    int32_t* G = static_cast<int32_t*>(ws);
    if (method == CCL_METHOD_UF) {
        const dim3 grid((W + cb::kBX - 1) / cb::kBX, (H + cb::kBY - 1) / cb::kBY, B);
        cb::k_uf_local<CONN><<<grid, dim3(cb::kBX, cb::kBY), 0, s>>>(img, H, W, npx, G);
        const int nrows = (H - 1) / cb::kBY, ncols = 2 * ((W + cb::kBX - 1) / cb::kBX);
        const long long per = (long long)nrows * W + (long long)ncols * H;
        if (per > 0) cb::k_uf_global<CONN><<<dim3(unsigned((per + 255) / 256), B), 256, 0, s>>>(img, H, W, npx, G, nrows, ncols, per);
        cb::k_link_flat<<<flat_blocks, 256, 0, s>>>(G, out, n, npx);
        return cudaGetLastError();
    }
    if (method == CCL_METHOD_LINE_UF) {
        const dim3 grid((W + cb::kLine - 1) / cb::kLine, H, B);
        cb::k_line_local<<<grid, cb::kLine, 0, s>>>(img, H, W, npx, G);
        cb::k_line_global<CONN><<<grid, cb::kLine, 0, s>>>(img, H, W, npx, G);
        cb::k_link_flat<<<flat_blocks, 256, 0, s>>>(G, out, n, npx);
        return cudaGetLastError();
    }
    // LE: iterate scan / analysis / relabel until a scan changes nothing
    int32_t* L = G;
    int32_t* R = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + align_up(size_t(n) * sizeof(int32_t)));
    int* changed = reinterpret_cast<int*>(reinterpret_cast<char*>(R) + align_up(size_t(n) * sizeof(int32_t)));
    cb::k_le_init<<<flat_blocks, 256, 0, s>>>(img, L, R, n, npx);
    const dim3 grid((W + cb::kBX - 1) / cb::kBX, (H + cb::kBY - 1) / cb::kBY, B);
    cudaError_t e;
    for (int it = 0;; ++it) {
        if ((e = cudaMemsetAsync(changed, 0, sizeof(int), s)) != cudaSuccess) return e;
        cb::k_le_scan<CONN><<<grid, dim3(cb::kBX, cb::kBY), 0, s>>>(L, R, H, W, npx, changed);
        int h = 0;
        if ((e = cudaMemcpyAsync(&h, changed, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
        if (!h) break;
        cb::k_le_analysis<<<flat_blocks, 256, 0, s>>>(L, R, n, npx);
        cb::k_le_relabel<<<flat_blocks, 256, 0, s>>>(L, R, n, npx);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    cb::k_le_out<<<flat_blocks, 256, 0, s>>>(L, out, n);
    return cudaGetLastError();
}

ccl_status_t validate_buffers(const Plan& p, const uint8_t* img, const int32_t* out, void* ws,
                              size_t ws_bytes, int stages) {
    const size_t n = size_t(p.g.B) * size_t(p.g.npx);
    if (n == 0) return CCL_OK;
    if ((stages & kK1) && !img) return CCL_ERR_NULL;
    if ((stages & kK3) && !out) return CCL_ERR_NULL;
    if (!ws) return CCL_ERR_NULL;
    if (ws_bytes < p.total()) return CCL_ERR_WORKSPACE;
    // 256-byte aligned (include/ccl.h): the kernels use 16-byte vector
    // accesses into the workspace regions, which are 256-byte multiples
    if (reinterpret_cast<uintptr_t>(ws) % kAlign) return CCL_ERR_WORKSPACE;
    if (img && out && overlaps(img, n, out, n * sizeof(int32_t))) return CCL_ERR_ALIAS;
    if (img && overlaps(img, n, ws, ws_bytes)) return CCL_ERR_ALIAS;
    if (out && overlaps(out, n * sizeof(int32_t), ws, ws_bytes)) return CCL_ERR_ALIAS;
    return CCL_OK;
}

ccl_status_t label_alloc(const uint8_t* images, int64_t B, int64_t H, int64_t W, int conn,
                         int32_t* out) {
    Plan p;
    ccl_status_t st = make_plan(B, H, W, conn, 0, p);
    if (st != CCL_OK) return st;
    if (B == 0) return CCL_OK;
    if (!images || !out) return CCL_ERR_NULL;
    const size_t n = size_t(B) * size_t(p.g.npx);
    if (overlaps(images, n, out, n * sizeof(int32_t))) return CCL_ERR_ALIAS;
    void* ws = nullptr;
    const size_t bytes = p.total();
    cudaError_t e = cudaMallocAsync(&ws, bytes, 0);
    if (e != cudaSuccess) return cuda_fail(e);
    st = run(p, conn, kAll, images, out, ws, 0);
    e = cudaFreeAsync(ws, 0);
    if (st == CCL_OK && e != cudaSuccess) return cuda_fail(e);
    return st;
}

}  // namespace

extern "C" {

#ifdef CCL_TIMELINE  // profiling builds only (not declared in include/ccl.h)
int ccl_debug_timeline(unsigned long long* out, int reset) {
    if (out && cudaMemcpyFromSymbol(out, ccl::g_tl, sizeof(unsigned long long) * 8) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long init[8];
        for (int i = 0; i < 8; ++i) init[i] = (i == 0 || i == 2 || i == 4 || i == 5) ? ~0ull : 0ull;
        if (cudaMemcpyToSymbol(ccl::g_tl, init, sizeof(init)) != cudaSuccess) return -1;
    }
    return 0;
}
#ifdef CCL_STATS
// per-K2-task counters (union steps, find hops, link retries, rounds) into a caller device buffer
int ccl_debug_k2_taskstat(unsigned* dev_buf) {
    return cudaMemcpyToSymbol(ccl::g_k2_taskstat, &dev_buf, sizeof(dev_buf)) == cudaSuccess ? 0 : -1;
}
#endif
// per-tile publish times (globaltimer) into a caller device buffer
int ccl_debug_tile_pub(unsigned long long* dev_buf) {
    return cudaMemcpyToSymbol(ccl::g_tile_pub, &dev_buf, sizeof(dev_buf)) == cudaSuccess ? 0 : -1;
}
// per-K2-task globaltimer (start, end) pairs into a caller device buffer (DBG 8 builds)
int ccl_debug_k2_stamps(unsigned long long* dev_buf) {
    return cudaMemcpyToSymbol(ccl::g_k2_stamps, &dev_buf, sizeof(dev_buf)) == cudaSuccess ? 0 : -1;
}
#endif

const char* ccl_status_string(ccl_status_t status) {
    switch (status) {
        case CCL_OK: return "ok";
        case CCL_ERR_NULL: return "a required pointer is NULL";
        case CCL_ERR_DIMS: return "invalid dimensions (need H >= 1, W >= 1, B >= 0)";
        case CCL_ERR_TOO_LARGE: return "image too large: H*W must be <= 2^31-1";
        case CCL_ERR_CONNECTIVITY: return "connectivity must be 4 or 8";
        case CCL_ERR_ALIAS: return "input and output/workspace buffers overlap";
        case CCL_ERR_WORKSPACE: return "workspace too small or misaligned";
        case CCL_ERR_CUDA: return "CUDA error (see ccl_last_cuda_error)";
        case CCL_ERR_CONFIG: return "unsupported tile configuration";
    }
    return "unknown status";
}

int ccl_last_cuda_error(void) { return g_last_cuda_error; }

size_t ccl_workspace_bytes(int64_t B, int64_t H, int64_t W, int connectivity) {
    Plan p;
    if (make_plan(B, H, W, connectivity, 0, p) != CCL_OK) return 0;
    return p.total();
}

ccl_status_t ccl_label(const uint8_t* image, int64_t H, int64_t W, int connectivity,
                       int32_t* labels_out) {
    return label_alloc(image, 1, H, W, connectivity, labels_out);
}

ccl_status_t ccl_label_batched(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                               int connectivity, int32_t* labels_out) {
    return label_alloc(images, B, H, W, connectivity, labels_out);
}

ccl_status_t ccl_label_batched_cfg_async(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                         int connectivity, int32_t* labels_out, void* workspace,
                                         size_t workspace_bytes, int tile_rows, void* stream) {
    Plan p;
    ccl_status_t st = make_plan(B, H, W, connectivity, tile_rows, p);
    if (st != CCL_OK) return st;
    if (B == 0) return CCL_OK;
    st = validate_buffers(p, images, labels_out, workspace, workspace_bytes, kAll);
    if (st != CCL_OK) return st;
    return run(p, connectivity, kAll, images, labels_out, workspace, static_cast<cudaStream_t>(stream));
}

ccl_status_t ccl_label_threshold_async(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                       int connectivity, int threshold, int32_t* labels_out, void* workspace,
                                       size_t workspace_bytes, int tile_rows, void* stream) {
    if (threshold < 0 || threshold > 255) return CCL_ERR_CONFIG;
    Plan p;
    ccl_status_t st = make_plan(B, H, W, connectivity, tile_rows, p);
    if (st != CCL_OK) return st;
    if (B == 0) return CCL_OK;
    st = validate_buffers(p, images, labels_out, workspace, workspace_bytes, kAll);
    if (st != CCL_OK) return st;
    p.g.thr = threshold;
    p.g.thr_k = (threshold <= 128 ? uint32_t(128 - threshold) : uint32_t(256 - threshold)) * 0x01010101u;
    return run(p, connectivity, kAll, images, labels_out, workspace, static_cast<cudaStream_t>(stream));
}

ccl_status_t ccl_label_batched_async(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                     int connectivity, int32_t* labels_out, void* workspace,
                                     size_t workspace_bytes, void* stream) {
    return ccl_label_batched_cfg_async(images, B, H, W, connectivity, labels_out, workspace,
                                       workspace_bytes, 0, stream);
}

// ----------------------------------------- the paper's comparison methods
// (kernels in ccl_baselines.cuh)
size_t ccl_method_workspace_bytes(int64_t B, int64_t H, int64_t W, int connectivity, int method) {
    if (method == CCL_METHOD_OPTIMIZED) return ccl_workspace_bytes(B, H, W, connectivity);
    if (check_geometry(B, H, W, connectivity) != CCL_OK) return 0;
    const size_t n = size_t(B) * size_t(H) * size_t(W);
    if (method == CCL_METHOD_UF || method == CCL_METHOD_LINE_UF) return align_up(n * sizeof(int32_t));
    if (method == CCL_METHOD_LE) return 2 * align_up(n * sizeof(int32_t)) + kAlign;
    return 0;
}

ccl_status_t ccl_label_equal_async(const uint8_t* images, int64_t B, int64_t H, int64_t W, int connectivity,
                                   int32_t* labels_out, void* workspace, size_t workspace_bytes, void* stream) {
    ccl_status_t st = check_geometry(B, H, W, connectivity);
    if (st != CCL_OK) return st;
    if (B == 0) return CCL_OK;
    if (B > 65535) return CCL_ERR_DIMS;
    if (!images || !labels_out || !workspace) return CCL_ERR_NULL;
    if (workspace_bytes < ccl_method_workspace_bytes(B, H, W, connectivity, CCL_METHOD_UF)) return CCL_ERR_WORKSPACE;
    const size_t n = size_t(B) * size_t(H) * size_t(W);
    if (overlaps(images, n, labels_out, n * 4) || overlaps(images, n, workspace, workspace_bytes) ||
        overlaps(labels_out, n * 4, workspace, workspace_bytes))
        return CCL_ERR_ALIAS;
    namespace cb = ccl::base;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const long long npx = (long long)H * W, nn = npx * B;
    int32_t* G = static_cast<int32_t*>(workspace);
    const dim3 grid(unsigned((W + cb::kBX - 1) / cb::kBX), unsigned((H + cb::kBY - 1) / cb::kBY), unsigned(B));
    const int nrows = int((H - 1) / cb::kBY), ncols = int(2 * ((W + cb::kBX - 1) / cb::kBX));
    const long long per = (long long)nrows * W + (long long)ncols * H;
    const unsigned flat_blocks = unsigned(std::min<long long>((nn + 255) / 256, (long long)sm_count() * 16));
    if (connectivity == 4) {
        cb::k_uf_local<4, true><<<grid, dim3(cb::kBX, cb::kBY), 0, s>>>(images, int(H), int(W), npx, G);
        if (per > 0)
            cb::k_uf_global<4, true><<<dim3(unsigned((per + 255) / 256), unsigned(B)), 256, 0, s>>>(
                images, int(H), int(W), npx, G, nrows, ncols, per);
    } else {
        cb::k_uf_local<8, true><<<grid, dim3(cb::kBX, cb::kBY), 0, s>>>(images, int(H), int(W), npx, G);
        if (per > 0)
            cb::k_uf_global<8, true><<<dim3(unsigned((per + 255) / 256), unsigned(B)), 256, 0, s>>>(
                images, int(H), int(W), npx, G, nrows, ncols, per);
    }
    cb::k_link_flat<<<flat_blocks, 256, 0, s>>>(G, labels_out, nn, npx, 0);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CCL_OK : cuda_fail(e);
}

size_t ccl_workspace_bytes_3d(int64_t B, int64_t D, int64_t H, int64_t W, int connectivity) {
    if (B < 0 || D < 1 || H < 1 || W < 1 || (connectivity != 6 && connectivity != 26)) return 0;
    if (H > INT32_MAX / W || H * W > INT32_MAX / D) return 0;
    return align_up(size_t(B) * size_t(D) * size_t(H) * size_t(W) * sizeof(int32_t));
}

ccl_status_t ccl_label_3d_async(const uint8_t* volumes, int64_t B, int64_t D, int64_t H, int64_t W,
                                int connectivity, int32_t* labels_out, void* workspace, size_t workspace_bytes,
                                void* stream) {
    if (B < 0 || D < 1 || H < 1 || W < 1) return CCL_ERR_DIMS;
    if (H > INT32_MAX / W || H * W > INT32_MAX / D) return CCL_ERR_TOO_LARGE;
    if (connectivity != 6 && connectivity != 26) return CCL_ERR_CONNECTIVITY;
    if (B == 0) return CCL_OK;
    namespace cv = ccl::vol;
    const long long bz = (D + cv::kZ - 1) / cv::kZ;
    if (B * bz > 65535 || B > 65535 || (H + cv::kY - 1) / cv::kY > 65535) return CCL_ERR_DIMS;  // grid limits
    if (!volumes || !labels_out || !workspace) return CCL_ERR_NULL;
    if (workspace_bytes < ccl_workspace_bytes_3d(B, D, H, W, connectivity)) return CCL_ERR_WORKSPACE;
    const long long nvox = D * H * W, n = nvox * B;
    if (overlaps(volumes, size_t(n), labels_out, size_t(n) * 4) || overlaps(volumes, size_t(n), workspace, workspace_bytes) ||
        overlaps(labels_out, size_t(n) * 4, workspace, workspace_bytes))
        return CCL_ERR_ALIAS;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int32_t* G = static_cast<int32_t*>(workspace);
    const dim3 grid(unsigned((W + cv::kX - 1) / cv::kX), unsigned((H + cv::kY - 1) / cv::kY), unsigned(B * bz));
    const dim3 blk(cv::kX, cv::kY, cv::kZ);
    const dim3 gb(unsigned((nvox + 255) / 256), unsigned(B));
    if (connectivity == 6) {
        cv::k_vol_local<6><<<grid, blk, 0, s>>>(volumes, int(D), int(H), int(W), nvox, int(bz), G);
        cv::k_vol_boundary<6><<<gb, 256, 0, s>>>(volumes, int(D), int(H), int(W), nvox, G);
    } else {
        cv::k_vol_local<26><<<grid, blk, 0, s>>>(volumes, int(D), int(H), int(W), nvox, int(bz), G);
        cv::k_vol_boundary<26><<<gb, 256, 0, s>>>(volumes, int(D), int(H), int(W), nvox, G);
    }
    const unsigned flat_blocks = unsigned(std::min<long long>((n + 255) / 256, (long long)sm_count() * 16));
    ccl::base::k_link_flat<<<flat_blocks, 256, 0, s>>>(G, labels_out, n, nvox, 1);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CCL_OK : cuda_fail(e);
}

ccl_status_t ccl_label_method_async(const uint8_t* images, int64_t B, int64_t H, int64_t W, int connectivity,
                                    int method, int32_t* labels_out, void* workspace, size_t workspace_bytes,
                                    void* stream) {
    if (method == CCL_METHOD_OPTIMIZED)
        return ccl_label_batched_async(images, B, H, W, connectivity, labels_out, workspace, workspace_bytes, stream);
    ccl_status_t st = check_geometry(B, H, W, connectivity);
    if (st != CCL_OK) return st;
    if (method != CCL_METHOD_UF && method != CCL_METHOD_LINE_UF && method != CCL_METHOD_LE) return CCL_ERR_CONFIG;
    if (B == 0) return CCL_OK;
    if (B > 65535 || H > 65535) return CCL_ERR_DIMS;  // grid.z = B, (line UF) grid.y = H
    if (!images || !labels_out || !workspace) return CCL_ERR_NULL;
    if (workspace_bytes < ccl_method_workspace_bytes(B, H, W, connectivity, method)) return CCL_ERR_WORKSPACE;
    const size_t n = size_t(B) * size_t(H) * size_t(W);
    if (overlaps(images, n, labels_out, n * 4) || overlaps(images, n, workspace, workspace_bytes) ||
        overlaps(labels_out, n * 4, workspace, workspace_bytes))
        return CCL_ERR_ALIAS;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const cudaError_t e = connectivity == 4 ? run_method<4>(method, images, int(B), int(H), int(W), labels_out, workspace, s)
                                            : run_method<8>(method, images, int(B), int(H), int(W), labels_out, workspace, s);
    return e == cudaSuccess ? CCL_OK : cuda_fail(e);
}

// ------------------------------------------- per-component statistics
size_t ccl_stats_workspace_bytes(int64_t B, int64_t H, int64_t W) {
    if (check_geometry(B, H, W, 8) != CCL_OK) return 0;
    const size_t npx = size_t(H) * size_t(W);
    const size_t nchunks = (npx + ccl::stats::kChunk - 1) / ccl::stats::kChunk;
    return align_up(size_t(B) * npx * sizeof(int32_t)) + align_up(size_t(B) * nchunks * sizeof(int32_t));
}

ccl_status_t ccl_component_stats_async(const int32_t* labels, int64_t B, int64_t H, int64_t W,
                                       int64_t max_components, ccl_component_t* stats, int32_t* counts,
                                       void* workspace, size_t workspace_bytes, void* stream) {
    return ccl_component_stats_relabel_async(labels, B, H, W, max_components, stats, counts, nullptr, workspace,
                                             workspace_bytes, stream);
}

ccl_status_t ccl_component_stats_relabel_async(const int32_t* labels, int64_t B, int64_t H, int64_t W,
                                               int64_t max_components, ccl_component_t* stats, int32_t* counts,
                                               int32_t* relabel_out, void* workspace, size_t workspace_bytes,
                                               void* stream) {
    ccl_status_t st = check_geometry(B, H, W, 8);
    if (st != CCL_OK) return st;
    if (max_components < 1 || B > 65535) return CCL_ERR_DIMS;
    if (B == 0) return CCL_OK;
    if (!labels || !stats || !counts || !workspace) return CCL_ERR_NULL;
    if (workspace_bytes < ccl_stats_workspace_bytes(B, H, W)) return CCL_ERR_WORKSPACE;
    const long long npx = (long long)H * W;
    const size_t nl = size_t(B) * size_t(npx) * 4, ns = size_t(B) * size_t(max_components) * sizeof(ccl_component_t);
    if (overlaps(labels, nl, stats, ns) || overlaps(labels, nl, workspace, workspace_bytes) ||
        overlaps(stats, ns, workspace, workspace_bytes) || overlaps(counts, size_t(B) * 4, stats, ns) ||
        overlaps(counts, size_t(B) * 4, workspace, workspace_bytes) || overlaps(counts, size_t(B) * 4, labels, nl))
        return CCL_ERR_ALIAS;
    if (relabel_out && (overlaps(relabel_out, nl, labels, nl) || overlaps(relabel_out, nl, stats, ns) ||
                        overlaps(relabel_out, nl, workspace, workspace_bytes) ||
                        overlaps(relabel_out, nl, counts, size_t(B) * 4)))
        return CCL_ERR_ALIAS;
    namespace cs = ccl::stats;
    const int nchunks = int((npx + cs::kChunk - 1) / cs::kChunk);
    int32_t* M = static_cast<int32_t*>(workspace);
    int32_t* cnt = reinterpret_cast<int32_t*>(static_cast<char*>(workspace) + align_up(size_t(B) * size_t(npx) * 4));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const dim3 gc(nchunks, unsigned(B));
    cs::k_stats_count<<<gc, cs::kT, 0, s>>>(labels, npx, nchunks, cnt);
    cs::k_stats_scan<<<unsigned(B), 1024, 0, s>>>(cnt, nchunks, counts);
    cs::k_stats_rank<<<gc, cs::kT, 0, s>>>(labels, npx, int(W), nchunks, cnt, M, stats, max_components);
    const unsigned ablocks = unsigned(std::max<long long>(1, std::min<long long>((npx + 16 * cs::kT - 1) / (16 * cs::kT),
                                                                                   std::max<long long>(1, (long long)sm_count() * 8 / B))));
    cs::k_stats_accum<<<dim3(ablocks, unsigned(B)), cs::kT, 0, s>>>(labels, npx, int(W), M, stats, max_components,
                                                                  relabel_out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CCL_OK : cuda_fail(e);
}

static ccl_status_t stage(const uint8_t* images, int64_t B, int64_t H, int64_t W, int conn,
                          int32_t* out, void* ws, size_t ws_bytes, int tile_rows, int which,
                          void* stream) {
    Plan p;
    ccl_status_t st = make_plan(B, H, W, conn, tile_rows, p);
    if (st != CCL_OK) return st;
    if (B == 0) return CCL_OK;
    st = validate_buffers(p, images, out, ws, ws_bytes, which);
    if (st != CCL_OK) return st;
    // the vector decision must match across stages: K1 decides on the image,
    // K3 on the output; both reduce to W % 16 == 0 for aligned buffers
    return run(p, conn, which, images, out, ws, static_cast<cudaStream_t>(stream));
}

ccl_status_t ccl_stage_local_merge(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                   int connectivity, void* workspace, size_t workspace_bytes,
                                   int tile_rows, void* stream) {
    return stage(images, B, H, W, connectivity, nullptr, workspace, workspace_bytes, tile_rows, kK1,
                 stream);
}

ccl_status_t ccl_stage_boundary(int64_t B, int64_t H, int64_t W, int connectivity, void* workspace,
                                size_t workspace_bytes, int tile_rows, void* stream) {
    return stage(nullptr, B, H, W, connectivity, nullptr, workspace, workspace_bytes, tile_rows, kK2,
                 stream);
}

ccl_status_t ccl_stage_link(int64_t B, int64_t H, int64_t W, int connectivity, int32_t* labels_out,
                            void* workspace, size_t workspace_bytes, int tile_rows, void* stream) {
    return stage(nullptr, B, H, W, connectivity, labels_out, workspace, workspace_bytes, tile_rows,
                 kK3, stream);
}

int ccl_default_tile_rows(int64_t B, int64_t H, int64_t W) {
    Plan p;
    if (make_plan(B, H, W, 4, 0, p) != CCL_OK) return -1;
    return p.ty;
}

int64_t ccl_boundary_work_items(int64_t B, int64_t H, int64_t W, int tile_rows,
                                int64_t* horizontal_segments, int64_t* vertical_pixels) {
    Plan p;
    if (make_plan(B, H, W, 4, tile_rows, p) != CCL_OK) return -1;
    const int64_t nh = B * int64_t(p.g.tiles_y - 1) * p.g.tiles_x;
    const int64_t nv = B * H * int64_t(p.g.tiles_x - 1);
    if (horizontal_segments) *horizontal_segments = nh;
    if (vertical_pixels) *vertical_pixels = nv;
    return nh + nv;
}

size_t ccl_host_scratch_bytes(int64_t B, int64_t H, int64_t W, int connectivity) {
    Plan p;
    if (make_plan(B, H, W, connectivity, 0, p) != CCL_OK) return 0;
    const size_t n = size_t(B) * size_t(p.g.npx);
    return align_up(n) + align_up(n * sizeof(int32_t)) + p.total();
}

ccl_status_t ccl_label_host_async(const uint8_t* h_images, int64_t B, int64_t H, int64_t W,
                                  int connectivity, int32_t* h_labels, void* d_scratch,
                                  size_t scratch_bytes, void* stream) {
    Plan p;
    ccl_status_t st = make_plan(B, H, W, connectivity, 0, p);
    if (st != CCL_OK) return st;
    if (B == 0) return CCL_OK;
    if (!h_images || !h_labels || !d_scratch) return CCL_ERR_NULL;
    if (scratch_bytes < ccl_host_scratch_bytes(B, H, W, connectivity)) return CCL_ERR_WORKSPACE;
    const size_t n = size_t(B) * size_t(p.g.npx);
    if (overlaps(h_images, n, h_labels, n * sizeof(int32_t))) return CCL_ERR_ALIAS;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* base = static_cast<char*>(d_scratch);
    uint8_t* d_img = reinterpret_cast<uint8_t*>(base);
    int32_t* d_out = reinterpret_cast<int32_t*>(base + align_up(n));
    void* ws = base + align_up(n) + align_up(n * sizeof(int32_t));
    cudaError_t e = cudaMemcpyAsync(d_img, h_images, n, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e);
    st = run(p, connectivity, kAll, d_img, d_out, ws, s);
    if (st != CCL_OK) return st;
    e = cudaMemcpyAsync(h_labels, d_out, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e);
    return CCL_OK;
}

// ------------------------------------------------------- strip sharding
static size_t align_up_c(size_t v) { return (v + 255) / 256 * 256; }

size_t ccl_strip_workspace_bytes(int64_t rows, int64_t W, int k, int connectivity) {
    Plan p;
    if (k < 1 || make_plan(1, rows, W, connectivity, 0, p) != CCL_OK) return 0;
    p.F_bytes = p.strip_F_bytes;
    return p.total() + align_up_c(size_t(k) * 2 * size_t(W) * sizeof(uint64_t));
}

static ccl_status_t strip_plan(int64_t rows, int64_t W, int64_t row0, int64_t H_total, int conn, int k,
                               int rank, Plan& p) {
    if (k < 1 || rank < 0 || rank >= k) return CCL_ERR_DIMS;
    if (rows < 1 || W < 1 || row0 < 0 || H_total < 1 || row0 + rows > H_total) return CCL_ERR_DIMS;
    if (H_total > INT32_MAX / W) return CCL_ERR_TOO_LARGE;  // labels are global raster indices
    if (int64_t(k) * 4 * W > INT32_MAX) return CCL_ERR_TOO_LARGE;
    ccl_status_t st = make_plan(1, rows, W, conn, 0, p);
    if (st != CCL_OK) return st;
    p.g.label_off = int(row0 * W);
    p.g.strip = 1;
    p.F_bytes = p.strip_F_bytes;
    p.g.force_top = row0 > 0;
    p.g.force_bottom = row0 + rows < H_total;
    return CCL_OK;
}

ccl_status_t ccl_strip_local(const uint8_t* strip, int64_t rows, int64_t W, int64_t row0, int64_t H_total,
                             int connectivity, int k, int32_t* send, int32_t* labels_out, void* workspace,
                             size_t workspace_bytes, void* stream) {
    Plan p;
    ccl_status_t st = strip_plan(rows, W, row0, H_total, connectivity, k, 0, p);
    if (st != CCL_OK) return st;
    if (!send) return CCL_ERR_NULL;
    st = validate_buffers(p, strip, labels_out, workspace, workspace_bytes, kAll);
    if (st != CCL_OK) return st;
    if (workspace_bytes < ccl_strip_workspace_bytes(rows, W, k, connectivity)) return CCL_ERR_WORKSPACE;
    StripCtx sc;
    sc.send = send;
    sc.k = k;
    sc.P = reinterpret_cast<uint64_t*>(static_cast<char*>(workspace) + p.total());
    return run(p, connectivity, kK1 | kK2 | kStripEdges, strip, labels_out, workspace,
               static_cast<cudaStream_t>(stream), &sc);
}

ccl_status_t ccl_strip_finalize(const int32_t* gathered, int k, int rank, int64_t rows, int64_t W, int64_t row0,
                                int64_t H_total, int connectivity, int32_t* labels_out, void* workspace,
                                size_t workspace_bytes, void* stream) {
    Plan p;
    ccl_status_t st = strip_plan(rows, W, row0, H_total, connectivity, k, rank, p);
    if (st != CCL_OK) return st;
    if (!gathered) return CCL_ERR_NULL;
    st = validate_buffers(p, nullptr, labels_out, workspace, workspace_bytes, kK3);
    if (st != CCL_OK) return st;
    if (workspace_bytes < ccl_strip_workspace_bytes(rows, W, k, connectivity)) return CCL_ERR_WORKSPACE;
    StripCtx sc;
    sc.gathered = gathered;
    sc.k = k;
    sc.rank = rank;
    sc.P = reinterpret_cast<uint64_t*>(static_cast<char*>(workspace) + p.total());
    return run(p, connectivity, kStripFinalize | kK3, nullptr, labels_out, workspace,
               static_cast<cudaStream_t>(stream), &sc);
}

}  // extern "C"
