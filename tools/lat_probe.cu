// tools/lat_probe.cu -- dependent-load latency on this GPU (profiling aid, not
// part of the library): one pointer chase per warp over a buffer of the given
// size, L2-resident (ld.global.cg) or L1-cacheable (ld.ca), with 1 .. many
// concurrent warps; reports ns per dependent load.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lat_probe.cu -o tools/lat_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s\n", cudaGetErrorString(e_)); exit(1); } } while (0)

template <int MODE>
__global__ void chase(const int* __restrict__ next, int start_stride, int steps, int* sink) {
    int p = (blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32) * start_stride;
    for (int i = 0; i < steps; ++i) {
        if (MODE == 0) p = __ldcg(next + p);
        else if (MODE == 1) { int v; asm volatile("ld.global.ca.s32 %0, [%1];" : "=r"(v) : "l"(next + p)); p = v; }
        else p = atomicAdd(const_cast<int*>(next) + p, 0);
    }
    if (p == -1) *sink = p;
}

int main() {
    const size_t n = size_t(16) << 20;  // 64 MB of ints
    std::vector<int> h(n);
    // random cyclic permutation at 32-B sector granularity (stride 8 ints)
    const size_t ns = n / 8;
    std::vector<int> perm(ns);
    for (size_t i = 0; i < ns; ++i) perm[i] = int(i);
    std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
    for (size_t i = 0; i < ns; ++i) h[size_t(perm[i]) * 8] = perm[(i + 1) % ns] * 8;
    int *d, *sink;
    CK(cudaMalloc(&d, n * 4));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int steps = 2000;
    for (int mode = 0; mode < 3; ++mode) {
        for (int warps : {1, 148, 1184, 4736, 9472}) {
            const int bs = 256, blocks = std::max(1, warps * 32 / bs), tb = warps * 32 < bs ? warps * 32 : bs;
            auto launch = [&] {
                if (mode == 0) chase<0><<<blocks, tb>>>(d, 997 * 8, steps, sink);
                else if (mode == 1) chase<1><<<blocks, tb>>>(d, 997 * 8, steps, sink);
                else chase<2><<<blocks, tb>>>(d, 997 * 8, steps, sink);
            };
            launch();
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%-10s warps %5d  %7.1f ns per dependent access\n", mode == 0 ? "ld.cg" : mode == 1 ? "ld.ca" : "atomicAdd",
                   warps, ms * 1e6 / steps);
        }
    }
    return 0;
}
