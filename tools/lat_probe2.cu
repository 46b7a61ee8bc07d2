// tools/lat_probe2.cu -- dependent-load latency under K2-like concurrency
// (profiling harness): W warps (one per task, all resident), each walks a
// chain of N dependent loads; the chain nodes lie in a region of R bytes
// (L2-resident when small; spread over many 2 MB pages when large).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/lat_probe2.cu -o tools/lat_probe2
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

template <int MODE>  // 0: ld.global.cg (L2), 1: ld.global.ca, 2: atomicAdd(0) returning
__global__ void chase(const uint32_t* __restrict__ nxt, uint32_t* out, int steps, size_t stride_words, unsigned long long* t) {
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    uint32_t p = uint32_t(((w * 7919u + lane * 104729u) % 4096u) * (stride_words / 4096));
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < steps; ++i) {
        uint32_t v;
        if (MODE == 0) v = __ldcg(nxt + p);
        else if (MODE == 1) asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(nxt + p));
        else v = atomicAdd(const_cast<uint32_t*>(nxt) + p, 0u);
        p = v;
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (lane == 0) t[w] = t1 - t0;
    if (p == 0xFFFFFFFFu) out[0] = p;
}

int main() {
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t maxbytes = size_t(512) << 20;
    uint32_t* buf; uint32_t* out; unsigned long long* t;
    CK(cudaMalloc(&buf, maxbytes)); CK(cudaMalloc(&out, 64)); CK(cudaMalloc(&t, 8 << 20));
    // sparse: 4096 nodes (one 32-B sector each, 128 KB of data, L2-resident)
    // spread over `region` bytes: the page count grows, the data does not
    for (size_t region : {size_t(4) << 20, size_t(64) << 20, size_t(512) << 20}) {
        const size_t nw = region / 4;
        std::vector<uint32_t> h(nw, 0);
        const size_t nodes = 4096, step = nw / nodes;
        uint64_t x = 12345;
        for (size_t i = 0; i < nodes; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i * step] = uint32_t((x % nodes) * step); }
        CK(cudaMemcpy(buf, h.data(), region, cudaMemcpyHostToDevice));
        for (int warps_per_sm : {1, 8, 40}) {
            const int nwarps = sms * warps_per_sm;
            for (int mode = 0; mode < 3; ++mode) {
                const int steps = 16;
                auto k = mode == 0 ? chase<0> : mode == 1 ? chase<1> : chase<2>;
                // warm-up (TLB / L2): one pass
                k<<<nwarps / 8 + 1, 256>>>(buf, out, steps, nw, t);
                CK(cudaDeviceSynchronize());
                k<<<nwarps / 8 + 1, 256>>>(buf, out, steps, nw, t);
                CK(cudaDeviceSynchronize());
                std::vector<unsigned long long> ht(nwarps);
                CK(cudaMemcpy(ht.data(), t, nwarps * 8, cudaMemcpyDeviceToHost));
                std::vector<double> d(ht.begin(), ht.end());
                std::sort(d.begin(), d.end());
                printf("region %4zu MB  warps/SM %2d  %s: per dependent load p50 %.0f ns  p90 %.0f ns  max %.0f ns\n",
                       region >> 20, warps_per_sm, mode == 0 ? "ld.cg     " : mode == 1 ? "ld.ca     " : "atomicAdd ",
                       d[d.size() / 2] / steps, d[d.size() * 9 / 10] / steps, d.back() / steps);
            }
        }
    }
    return 0;
}
