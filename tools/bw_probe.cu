// tools/bw_probe.cu -- HBM read / write floors on B200 for the access shapes
// the CCL kernels can use (profiling harness, not part of libccl.so).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/bw_probe.cu -o tools/bw_probe
// Reads: 64 MiB (C3 image); writes: 256 MiB (C3 labels); L2 flushed (512 MiB
// memset) before every timed launch; CUDA events; mean of 20.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
            exit(1);                                                                     \
        }                                                                                \
    } while (0)

__device__ __forceinline__ uint4 ld_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
struct U8 { uint32_t v[8]; };
__device__ __forceinline__ U8 ld_v8(const void* p) {
    U8 r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                   "=r"(r.v[6]), "=r"(r.v[7]) : "l"(p));
    return r;
}

// R1: 4 independent 16-B loads per thread per iteration
__global__ void r_v4x4(const uint4* p, size_t n, unsigned* sink) {
    unsigned acc = 0;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i + 3 * stride < n; i += 4 * stride) {
        uint4 a = ld_v4(p + i), b = ld_v4(p + i + stride), c = ld_v4(p + i + 2 * stride), d = ld_v4(p + i + 3 * stride);
        acc ^= a.x ^ b.y ^ c.z ^ d.w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}
// R2: 2 independent 32-B loads per thread per iteration
__global__ void r_v8x2(const uint8_t* p, size_t n32, unsigned* sink) {
    unsigned acc = 0;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i + stride < n32; i += 2 * stride) {
        U8 a = ld_v8(p + 32 * i), b = ld_v8(p + 32 * (i + stride));
        acc ^= a.v[0] ^ b.v[7];
    }
    if (acc == 0x12345678u) sink[0] = acc;
}
// R3: bulk copies (cp.async.bulk, non-tensor) of 16 KB chunks into shared
// memory, NBUF buffers per block, one thread issues, mbarrier completion
template <int NBUF>
__global__ void r_bulk(const uint8_t* p, size_t nchunks, unsigned* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[NBUF];
    constexpr unsigned CH = 16384;
    if (threadIdx.x == 0)
        for (int b = 0; b < NBUF; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(unsigned(__cvta_generic_to_shared(&bar[b]))));
    __syncthreads();
    unsigned acc = 0;
    size_t c = blockIdx.x;
    int it = 0;
    auto issue = [&](size_t ch, int b) {
        const unsigned ba = unsigned(__cvta_generic_to_shared(&bar[b]));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(CH) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         unsigned(__cvta_generic_to_shared(sm + b * CH))),
                     "l"(p + ch * CH), "r"(CH), "r"(ba)
                     : "memory");
    };
    if (threadIdx.x == 0)
        for (int b = 0; b < NBUF; ++b)
            if (c + size_t(b) * gridDim.x < nchunks) issue(c + size_t(b) * gridDim.x, b);
    for (; c < nchunks; c += gridDim.x, ++it) {
        const int b = it % NBUF;
        const unsigned ph = (it / NBUF) & 1;
        const unsigned ba = unsigned(__cvta_generic_to_shared(&bar[b]));
        asm volatile(
            "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}" ::"r"(ba),
            "r"(ph)
            : "memory");
        const uint4 v = reinterpret_cast<const uint4*>(sm + b * CH)[threadIdx.x];
        acc ^= v.x;
        __syncthreads();
        if (threadIdx.x == 0 && c + size_t(NBUF) * gridDim.x < nchunks) issue(c + size_t(NBUF) * gridDim.x, b);
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void w_v4cs(int32_t* p, size_t n4) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x)
        asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p + 4 * i), "r"(int(i)), "r"(0), "r"(1), "r"(2)
                     : "memory");
}
__global__ void w_v4(int32_t* p, size_t n4) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x)
        asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p + 4 * i), "r"(int(i)), "r"(0), "r"(1), "r"(2)
                     : "memory");
}
__global__ void w_v8cs(int32_t* p, size_t n8) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n8; i += size_t(gridDim.x) * blockDim.x)
        asm volatile("st.global.cs.v8.s32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p + 8 * i), "r"(int(i)), "r"(0),
                     "r"(1), "r"(2), "r"(3), "r"(4), "r"(5), "r"(6)
                     : "memory");
}
__global__ void w_v8(int32_t* p, size_t n8) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n8; i += size_t(gridDim.x) * blockDim.x)
        asm volatile("st.global.v8.s32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p + 8 * i), "r"(int(i)), "r"(0),
                     "r"(1), "r"(2), "r"(3), "r"(4), "r"(5), "r"(6)
                     : "memory");
}
// bulk S2G stores of CH-byte chunks from shared memory (one thread issues;
// the block's threads refill a buffer once its previous store has been read)
template <unsigned CH, int NBUF>
__global__ void w_bulk(int32_t* p, size_t nchunks) {
    extern __shared__ __align__(128) uint8_t sm[];
    int it = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int b = it % NBUF;
        if (threadIdx.x == 0 && it >= NBUF) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
        __syncthreads();
        int4* d = reinterpret_cast<int4*>(sm + b * CH);
        for (unsigned j = threadIdx.x; j < CH / 16; j += blockDim.x) d[j] = make_int4(int(c), int(j), 1, 2);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                             reinterpret_cast<char*>(p) + c * CH),
                         "r"(unsigned(__cvta_generic_to_shared(sm + b * CH))), "r"(CH)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// K3's store pattern without its compute: persistent blocks of 8 warps walk
// 1024 x 16 int32 tiles (t = block, block + grid, ...); each warp stores its
// two 4 KB rows of a tile with bulk S2G copies from its own smem row buffer
// (waiting for the previous store to have read the buffer first).
template <int ROWS_PER_STORE>
__global__ void w_k3pattern(int32_t* out, int H, int W, unsigned ntiles) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int4* buf = reinterpret_cast<int4*>(sm + warp * 4096 * ROWS_PER_STORE);
    const int tiles_x = W / 1024;
    for (unsigned t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tx = t % tiles_x, ty = t / tiles_x;
        for (int r = warp * ROWS_PER_STORE; r < 16; r += 8 * ROWS_PER_STORE) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            for (int q = lane; q < 256 * ROWS_PER_STORE; q += 32) buf[q] = make_int4(int(t), r, q, 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                for (int rr = 0; rr < ROWS_PER_STORE; ++rr) {
                    int32_t* dst = out + size_t(ty * 16 + r + rr) * W + tx * 1024;
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                                 "r"(unsigned(__cvta_generic_to_shared(buf + 256 * rr))), "r"(4096u)
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void copy_v4(const uint4* a, uint4* b, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        b[i] = a[i];
}

void* g_flush;
const size_t kFlush = size_t(512) << 20;

template <typename F>
float timeit(F f, int iters = 20) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float tot = 0;
    for (int i = 0; i < iters + 3; ++i) {
        CK(cudaMemsetAsync(g_flush, i, kFlush));
        CK(cudaEventRecord(a));
        f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (i >= 3) tot += ms;
    }
    CK(cudaGetLastError());
    return 1000.f * tot / iters;
}

int main() {
    const size_t nr = size_t(64) << 20, nw = size_t(256) << 20;
    uint8_t* img;
    int32_t* out;
    unsigned* sink;
    CK(cudaMalloc(&img, nr));
    CK(cudaMalloc(&out, nw));
    CK(cudaMalloc(&sink, 64));
    CK(cudaMalloc(&g_flush, kFlush));
    CK(cudaMemset(img, 1, nr));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    auto rep = [](const char* nm, float us, size_t bytes) { printf("%-44s %8.2f us  %7.1f GB/s\n", nm, us, bytes / us / 1e3); };
    for (int per : {4, 8, 16}) {
        char nm[80];
        snprintf(nm, sizeof nm, "read v4 x4 in flight, %d blk/SM", per);
        rep(nm, timeit([&] { r_v4x4<<<sms * per, 256>>>(reinterpret_cast<const uint4*>(img), nr / 16, sink); }), nr);
        snprintf(nm, sizeof nm, "read v8 x2 in flight, %d blk/SM", per);
        rep(nm, timeit([&] { r_v8x2<<<sms * per, 256>>>(img, nr / 32, sink); }), nr);
    }
    {
        auto k = r_bulk<2>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16384));
        for (int per : {2, 4, 6})
        {
            char nm[80];
            snprintf(nm, sizeof nm, "read bulk 16KB x2 buf, %d blk/SM", per);
            rep(nm, timeit([&] { k<<<sms * per, 1024 / 1, 2 * 16384>>>(img, nr / 16384, sink); }), nr);
        }
        auto k4 = r_bulk<4>;
        CK(cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
        for (int per : {1, 2, 3}) {
            char nm[80];
            snprintf(nm, sizeof nm, "read bulk 16KB x4 buf, %d blk/SM", per);
            rep(nm, timeit([&] { k4<<<sms * per, 1024, 4 * 16384>>>(img, nr / 16384, sink); }), nr);
        }
    }
    for (int per : {3, 4, 8, 16}) {
        char nm[80];
        snprintf(nm, sizeof nm, "write v4.cs, %d blk/SM", per);
        rep(nm, timeit([&] { w_v4cs<<<sms * per, 256>>>(out, nw / 16); }), nw);
        snprintf(nm, sizeof nm, "write v4 (wb), %d blk/SM", per);
        rep(nm, timeit([&] { w_v4<<<sms * per, 256>>>(out, nw / 16); }), nw);
        snprintf(nm, sizeof nm, "write v8.cs, %d blk/SM", per);
        rep(nm, timeit([&] { w_v8cs<<<sms * per, 256>>>(out, nw / 32); }), nw);
        snprintf(nm, sizeof nm, "write v8 (wb), %d blk/SM", per);
        rep(nm, timeit([&] { w_v8<<<sms * per, 256>>>(out, nw / 32); }), nw);
    }
    {
        auto k1 = w_bulk<4096, 4>;
        auto k2 = w_bulk<16384, 2>;
        auto k3 = w_bulk<16384, 4>;
        CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4096));
        CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16384));
        CK(cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
        for (int per : {2, 4, 8}) {
            char nm[80];
            snprintf(nm, sizeof nm, "write bulk 4KB x4, %d blk/SM", per);
            rep(nm, timeit([&] { k1<<<sms * per, 256, 4 * 4096>>>(out, nw / 4096); }), nw);
            snprintf(nm, sizeof nm, "write bulk 16KB x2, %d blk/SM", per);
            rep(nm, timeit([&] { k2<<<sms * per, 256, 2 * 16384>>>(out, nw / 16384); }), nw);
            if (per <= 3 || per == 2) {
                snprintf(nm, sizeof nm, "write bulk 16KB x4, %d blk/SM", per);
                rep(nm, timeit([&] { k3<<<sms * per, 256, 4 * 16384>>>(out, nw / 16384); }), nw);
            }
        }
    }
    {
        const int H = 8192, W = 8192;
        const unsigned ntiles = (H / 16) * (W / 1024);
        auto k1 = w_k3pattern<1>;
        auto k2 = w_k3pattern<2>;
        CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096));
        CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192));
        for (int per : {3, 4, 6}) {
            char nm[80];
            snprintf(nm, sizeof nm, "write K3 pattern 4KB rows, %d blk/SM", per);
            rep(nm, timeit([&] { k1<<<sms * per, 256, 8 * 4096>>>(out, H, W, ntiles); }), nw);
            snprintf(nm, sizeof nm, "write K3 pattern 2x4KB per store, %d blk/SM", per);
            rep(nm, timeit([&] { k2<<<sms * per, 256, 8 * 8192>>>(out, H, W, ntiles); }), nw);
        }
    }
    rep("copy v4 (256 MiB -> 256 MiB, r+w bytes)", timeit([&] {
            copy_v4<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(out), reinterpret_cast<uint4*>(g_flush), nw / 16);
        }), 2 * nw);
    return 0;
}
