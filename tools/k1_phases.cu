// tools/k1_phases.cu -- profiling harness (not part of libccl.so): times the
// K1 local-merge kernel with phases disabled (DBG template bits) and the HBM
// read / write floors on the same image, to locate where K1/K3 time goes.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include \
//        tools/k1_phases.cu -o tools/k1_phases
//   tools/k1_phases <raw uint8 image file> H W [conn]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CCL_K2_PHASES 1
#include "../paper_1708_08180_b200/csrc/ccl_kernels.cuh"
#include <cudaTypedefs.h>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__global__ void read_floor(const uint4* p, size_t n, unsigned* sink) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        uint4 v = ccl::ld_stream_u4(reinterpret_cast<const uint8_t*>(p + i));
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void write_floor(int32_t* p, size_t n4) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x)
        ccl::st_stream_i4(p + 4 * i, int(i), 0, 1, 2);
}

// Touch K1's outputs (mask, the used part of every tile's run records, edge
// blocks, the edge roots' parent sectors) so they are L2-resident: isolates
// how much of K2's time is DRAM latency on K1's outputs.
__global__ void touch_k1_outputs(const uint32_t* bits, size_t nwords, const uint32_t* R, int rcap,
                                 const int32_t* E, const uint64_t* G, unsigned ntiles, unsigned* sink) {
    unsigned acc = 0;
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x, nt = size_t(gridDim.x) * blockDim.x;
    for (size_t i = tid; i < nwords; i += nt) acc ^= __ldcg(bits + i);
    for (size_t i = tid; i < size_t(ntiles) * 512; i += nt) acc ^= __ldcg(R + (i / 512) * rcap + (i % 512));
    for (size_t t = tid; t < ntiles; t += nt) {
        const int32_t* Et = E + t * ccl::kEdgeCap;
        const int n = __ldcg(Et);
        for (int j = 0; j < ccl::kEdgeCap; ++j) acc ^= __ldcg(Et + j);
        for (int j = 0; j < n; ++j) acc ^= unsigned(__ldcg(reinterpret_cast<const unsigned long long*>(G) + ccl::edge_slot(ntiles, j, unsigned(t))));
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

template <typename F>
float timeit(F f, void* flush, size_t flush_bytes, int iters = 20) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float tot = 0;
    for (int i = 0; i < iters + 3; ++i) {
        CK(cudaMemsetAsync(flush, i, flush_bytes));
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

static int32_t* g_F = nullptr;
template <int TY, int CONN, int DBG>
void run_k1(const char* name, const uint8_t* img, ccl::Geom g, uint32_t* bits, uint64_t* G, uint32_t* R,
            int32_t* E, unsigned ntiles, int grid, void* flush, size_t fb) {
    auto k = ccl::k_local_merge<TY, CONN, true, DBG>;
    size_t smem = sizeof(ccl::K1Smem<TY>);
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    float us = timeit([&] { k<<<grid, ccl::k1_threads<TY>(), smem>>>(img, g, bits, G, R, E, g_F, ntiles); }, flush, fb);
    printf("%-34s grid %6d  %8.1f us\n", name, grid, us);
}

int main(int argc, char** argv) {
    if (argc < 4) {
        fprintf(stderr, "usage: %s image.raw H W [conn]\n", argv[0]);
        return 2;
    }
    const int H = atoi(argv[2]), W = atoi(argv[3]);
    const size_t n = size_t(H) * W;
    std::vector<uint8_t> h(n);
    FILE* f = fopen(argv[1], "rb");
    if (!f || fread(h.data(), 1, n, f) != n) {
        fprintf(stderr, "cannot read image\n");
        return 2;
    }
    fclose(f);
    uint8_t* img;
    uint64_t* G;
    int32_t* out;
    uint32_t* bits;
    uint32_t* R;
    int32_t *E, *F;
    void* flush;
    const size_t fb = size_t(512) << 20;
    CK(cudaMalloc(&img, n));
    CK(cudaMalloc(&G, (n / 1024 / 8 + 64) * ccl::edge_slots(8) * 8 * 4));
    CK(cudaMalloc(&out, n * 4));
    CK(cudaMalloc(&bits, n / 8 + 4096));
    CK(cudaMalloc(&R, 2 * n + 65536));
    CK(cudaMalloc(&E, (n / 1024 / 8 + 64) * ccl::kEdgeCap * 4));
    CK(cudaMalloc(&F, (n / 1024 / 8 + 64) * ccl::edge_slots(8) * 4 * 4));
    g_F = F;
    CK(cudaMalloc(&flush, fb));
    unsigned* sink;
    CK(cudaMalloc(&sink, 64));
    CK(cudaMemcpy(img, h.data(), n, cudaMemcpyHostToDevice));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));

    float r = timeit([&] { read_floor<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(img), n / 16, sink); }, flush, fb);
    printf("%-34s %8.1f us  %7.1f GB/s\n", "read floor (image, 1 B/px)", r, n / r / 1e3);
    float w = timeit([&] { write_floor<<<sms * 8, 256>>>(out, n / 4); }, flush, fb);
    printf("%-34s %8.1f us  %7.1f GB/s\n", "write floor (labels, 4 B/px)", w, 4 * n / w / 1e3);

#ifndef KP_TY
#define KP_TY 16
#endif
    constexpr int TY = KP_TY;
    ccl::Geom g;
    g.B = 1;
    g.H = H;
    g.W = W;
    g.WW = (W + 31) / 32;
    g.tiles_x = (W + 1023) / 1024;
    g.tiles_y = (H + TY - 1) / TY;
    g.npx = n;
    g.nwords = size_t(H) * g.WW;
    const unsigned ntiles = g.tiles_x * g.tiles_y;
    g.div_tx = ccl::FastDiv(g.tiles_x);
    g.div_ty = ccl::FastDiv(g.tiles_y);
    g.div_ty1 = ccl::FastDiv(std::max(1, g.tiles_y - 1));
    g.div_tx1 = ccl::FastDiv(std::max(1, g.tiles_x - 1));
    g.div_vg = ccl::FastDiv((g.tiles_y + 32 / TY - 1) / (32 / TY));
    g.label_off = g.force_top = g.force_bottom = 0;
    g.k3_early = 1;
    g.ntiles = ntiles;
    g.epoch = 0;
    g.ready = nullptr;
    g.strip = 0;
    CK(cudaMalloc(&g.defer, size_t(ntiles) * 4 + 4096));
    for (int per_sm : {4, 5}) {
        int grid = std::min<int>(ntiles, sms * per_sm);
        char nm[64];
        snprintf(nm, sizeof nm, "K1 load+convert+runs (DBG=3) x%d", per_sm);
        run_k1<TY, 8, 3>(nm, img, g, bits, G, R, E, ntiles, grid, flush, fb);
        snprintf(nm, sizeof nm, "K1 +UF loop, no unions (DBG=10) x%d", per_sm);
        run_k1<TY, 8, 10>(nm, img, g, bits, G, R, E, ntiles, grid, flush, fb);
        snprintf(nm, sizeof nm, "K1 +UF one atomic each (DBG=18) x%d", per_sm);
        run_k1<TY, 8, 18>(nm, img, g, bits, G, R, E, ntiles, grid, flush, fb);
        snprintf(nm, sizeof nm, "K1 +local UF (DBG=2) x%d", per_sm);
        run_k1<TY, 8, 2>(nm, img, g, bits, G, R, E, ntiles, grid, flush, fb);
        snprintf(nm, sizeof nm, "K1 full (DBG=0) x%d", per_sm);
        run_k1<TY, 8, 0>(nm, img, g, bits, G, R, E, ntiles, grid, flush, fb);
    }
    run_k1<TY, 8, 0>("K1 full, one block per tile", img, g, bits, G, R, E, ntiles, ntiles, flush, fb);

    // per-phase clock64 stamps (DBG bit 2), persistent grid x5
    unsigned long long* st;
    CK(cudaMalloc(&st, size_t(ntiles) * 8 * 8));
    CK(cudaMemset(st, 0, size_t(ntiles) * 8 * 8));
    CK(cudaMemcpyToSymbol(ccl::g_k1_stamps, &st, sizeof(st)));
    run_k1<TY, 8, 4>("K1 full + stamps x5", img, g, bits, G, R, E, ntiles, std::min<int>(ntiles, sms * 5), flush, fb);
    std::vector<unsigned long long> hs(size_t(ntiles) * 8);
    CK(cudaMemcpy(hs.data(), st, hs.size() * 8, cudaMemcpyDeviceToHost));
    const char* names[6] = {"convert+row init", "run lists", "union", "flatten", "edges+G", "run records"};
    double acc[6] = {0};
    for (unsigned t = 0; t < ntiles; ++t)
        for (int k = 0; k < 6; ++k) acc[k] += double(hs[t * 8 + k + 1] - hs[t * 8 + k]);
    double tot = 0;
    for (int k = 0; k < 6; ++k) tot += acc[k];
    printf("per-tile phase cycles (mean over %u tiles):\n", ntiles);
    for (int k = 0; k < 6; ++k) printf("  %-18s %8.0f  (%4.1f%%)\n", names[k], acc[k] / ntiles, 100 * acc[k] / tot);
    printf("  %-18s %8.0f\n", "total", tot / ntiles);

    // K2 variants (each preceded by K1, which resets the G entries K2 touches)
    auto k1 = ccl::k_local_merge<TY, 8, true, 0>;
    const int grid1 = std::min<int>(ntiles, sms * 5);
    const size_t sm1 = sizeof(ccl::K1Smem<TY>);
    const long long n_h = (long long)(g.tiles_y - 1) * g.tiles_x, n_v = (long long)((g.tiles_y + ccl::v_bands<TY>() - 1) / ccl::v_bands<TY>()) * (g.tiles_x - 1);
    const long long bh = (n_h + n_v + 7) / 8, bv = 0;
    auto time_k2 = [&](auto k2, const char* nm) {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        float tot2 = 0;
        for (int i = 0; i < 23; ++i) {
            CK(cudaMemsetAsync(flush, i, fb));
            k1<<<grid1, ccl::k1_threads<TY>(), sm1>>>(img, g, bits, G, R, E, F, ntiles);
            CK(cudaEventRecord(a));
            k2<<<unsigned(bh + bv), 256>>>(g, bits, R, E, G, n_h, n_v, 0);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (i >= 3) tot2 += ms;
        }
        printf("%-34s %8.1f us\n", nm, 1000.f * tot2 / 20);
    };
    time_k2(ccl::k_boundary<TY, 8, 0>, "K2 full");
    CK(cudaFuncSetAttribute(ccl::k_boundary<TY, 8, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 40));
    time_k2(ccl::k_boundary<TY, 8, 0>, "K2 full (carveout 40)");

    time_k2(ccl::k_boundary<TY, 8, 1>, "K2 horizontal only");
    time_k2(ccl::k_boundary<TY, 8, 2>, "K2 vertical only");
    time_k2(ccl::k_boundary<TY, 8, 3>, "K2 empty (launch)");
    time_k2(ccl::k_boundary<TY, 8, 5>, "K2 horizontal, no unions");
    {
        // K2 with K1's outputs pulled into L2 first (touch kernel outside the events)
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        float tot2 = 0;
        for (int i = 0; i < 23; ++i) {
            CK(cudaMemsetAsync(flush, i, fb));
            k1<<<grid1, ccl::k1_threads<TY>(), sm1>>>(img, g, bits, G, R, E, F, ntiles);
            touch_k1_outputs<<<sms * 4, 256>>>(bits, g.nwords, R, ccl::runs_per_tile_cap<TY>(), E, G, ntiles, sink);
            CK(cudaEventRecord(a));
            ccl::k_boundary<TY, 8, 0><<<unsigned(bh + bv), 256>>>(g, bits, R, E, G, n_h, n_v, 0);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (i >= 3) tot2 += ms;
        }
        printf("%-34s %8.1f us\n", "K2 full, K1 outputs L2-resident", 1000.f * tot2 / 20);
    }
    {
        // per-task K2 timeline (globaltimer): where does the kernel's time go?
        const long long nt = n_h + n_v;
        unsigned long long* st2;
        CK(cudaMalloc(&st2, size_t(nt) * 16));
        CK(cudaMemcpyToSymbol(ccl::g_k2_stamps, &st2, sizeof(st2)));
        CK(cudaMemsetAsync(flush, 1, fb));
        unsigned long long* ph;
        CK(cudaMalloc(&ph, size_t(nt) * 32));
        for (int ver = 0; ver < 1; ++ver) {
        CK(cudaMemset(ph, 0, size_t(nt) * 32));
        if (ver == 0) CK(cudaMemcpyToSymbol(ccl::g_k2_phase, &ph, sizeof(ph)));
        k1<<<grid1, ccl::k1_threads<TY>(), sm1>>>(img, g, bits, G, R, E, F, ntiles);
        auto kt = ccl::k_boundary<TY, 8, 8>;
        kt<<<unsigned(bh + bv), 256>>>(g, bits, R, E, G, n_h, n_v, 0);
        CK(cudaDeviceSynchronize());
        printf("[%s] ", ver == 0 ? "K2" : "K2v2");
        if (ver == 0) {
            unsigned long long* z = nullptr;
            CK(cudaMemcpyToSymbol(ccl::g_k2_phase, &z, sizeof(z)));
            std::vector<unsigned long long> hp(size_t(nt) * 4), hs0(size_t(nt) * 2);
            CK(cudaMemcpy(hp.data(), ph, hp.size() * 8, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(hs0.data(), st2, hs0.size() * 8, cudaMemcpyDeviceToHost));
            std::vector<double> d0, d1, d2, d3;
            for (long long i = 0; i < n_h; ++i) {
                if (!hp[4 * i] || !hp[4 * i + 1] || !hp[4 * i + 2]) continue;
                d0.push_back((hp[4 * i] - hs0[2 * i]) / 1000.0);
                d1.push_back((hp[4 * i + 1] - hp[4 * i]) / 1000.0);
                d2.push_back((hp[4 * i + 2] - hp[4 * i + 1]) / 1000.0);
                d3.push_back((hs0[2 * i + 1] - hp[4 * i + 2]) / 1000.0);
            }
            auto pc = [](std::vector<double> v, double q) { std::sort(v.begin(), v.end()); return v.empty() ? 0.0 : v[size_t(q * (v.size() - 1))]; };
            printf("K2 horizontal phases (us, p50/p90/max): masks-in %.2f/%.2f/%.2f  records-in %.2f/%.2f/%.2f  1st batch %.2f/%.2f/%.2f  rest %.2f/%.2f/%.2f  (n=%zu)\n",
                   pc(d0, .5), pc(d0, .9), pc(d0, 1), pc(d1, .5), pc(d1, .9), pc(d1, 1), pc(d2, .5), pc(d2, .9), pc(d2, 1),
                   pc(d3, .5), pc(d3, .9), pc(d3, 1), d0.size());
        }
        std::vector<unsigned long long> hs(size_t(nt) * 2);
        CK(cudaMemcpy(hs.data(), st2, hs.size() * 8, cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull, t1 = 0;
        for (long long i = 0; i < nt; ++i) { t0 = std::min(t0, hs[2 * i]); t1 = std::max(t1, hs[2 * i + 1]); }
        printf("K2 timeline: span %.1f us over %lld tasks\n", (t1 - t0) / 1000.0, nt);
        for (int kind = 0; kind < 2; ++kind) {
            std::vector<double> d, st, en;
            for (long long i = kind ? n_h : 0; i < (kind ? nt : n_h); ++i) {
                d.push_back((hs[2 * i + 1] - hs[2 * i]) / 1000.0);
                st.push_back((hs[2 * i] - t0) / 1000.0);
                en.push_back((hs[2 * i + 1] - t0) / 1000.0);
            }
            if (d.empty()) continue;
            auto pct = [](std::vector<double> v, double q) { std::sort(v.begin(), v.end()); return v[size_t(q * (v.size() - 1))]; };
            printf("  %s: dur p50 %.2f p90 %.2f p99 %.2f max %.2f | start p50 %.2f max %.2f | end p50 %.2f p99 %.2f max %.2f us\n",
                   kind ? "vertical  " : "horizontal", pct(d, .5), pct(d, .9), pct(d, .99), pct(d, 1.0), pct(st, .5),
                   pct(st, 1.0), pct(en, .5), pct(en, .99), pct(en, 1.0));
        }
        }
#ifdef CCL_STATS
        {   // the slowest tasks: what do they do?
            unsigned* ts;
            CK(cudaMalloc(&ts, size_t(nt) * 16));
            CK(cudaMemset(ts, 0, size_t(nt) * 16));
            CK(cudaMemcpyToSymbol(ccl::g_k2_taskstat, &ts, sizeof(ts)));
            k1<<<grid1, ccl::k1_threads<TY>(), sm1>>>(img, g, bits, G, R, E, F, ntiles);
            ccl::k_boundary<TY, 8, 0><<<unsigned(bh + bv), 256>>>(g, bits, R, E, G, n_h, n_v);
            CK(cudaDeviceSynchronize());
            std::vector<unsigned> hts(size_t(nt) * 4);
            CK(cudaMemcpy(hts.data(), ts, hts.size() * 4, cudaMemcpyDeviceToHost));
            std::vector<long long> idx(nt);
            for (long long i = 0; i < nt; ++i) idx[i] = i;
            std::sort(idx.begin(), idx.end(), [&](long long x, long long y) { return hts[4 * x] > hts[4 * y]; });
            double sst = 0, sho = 0, sre = 0, sro = 0;
            for (long long i = 0; i < nt; ++i) { sst += hts[4*i]; sho += hts[4*i+1]; sre += hts[4*i+2]; sro += hts[4*i+3]; }
            printf("K2 per task mean: steps %.1f hops %.1f retries %.2f rounds %.2f\n", sst / nt, sho / nt, sre / nt, sro / nt);
            for (int k = 0; k < 12 && k < nt; ++k) {
                const long long i = idx[k];
                printf("  busiest task %lld (%s): steps %u hops %u retries %u rounds %u\n", i, i < n_h ? "h" : "v",
                       hts[4*i], hts[4*i+1], hts[4*i+2], hts[4*i+3]);
            }
            unsigned* np2 = nullptr;
            CK(cudaMemcpyToSymbol(ccl::g_k2_taskstat, &np2, sizeof(np2)));
            CK(cudaFree(ts));
        }
#endif
        CK(cudaFree(st2));
        unsigned long long* np = nullptr;
        CK(cudaMemcpyToSymbol(ccl::g_k2_stamps, &np, sizeof(np)));
    }
    {
        k1<<<grid1, ccl::k1_threads<TY>(), sm1>>>(img, g, bits, G, R, E, F, ntiles);
        ccl::k_boundary<TY, 8, 0><<<unsigned(bh + bv), 256>>>(g, bits, R, E, G, n_h, n_v);
        float us = timeit([&] { ccl::k_resolve<TY><<<std::min<unsigned>((ntiles + 7) / 8, 148 * 16), 256>>>(g, G, E, F, ntiles); }, flush, fb);
        printf("%-34s %8.1f us\n", "K2b resolve", us);
    }

#ifdef CCL_STATS
    {
        unsigned long long z = 0, u, st, nf, nh, mh;
        CK(cudaMemcpyToSymbol(ccl::g_stat_unions, &z, 8));
        CK(cudaMemcpyToSymbol(ccl::g_stat_steps, &z, 8));
        k1<<<grid1, ccl::k1_threads<TY>(), sm1>>>(img, g, bits, G, R, E, F, ntiles);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpyToSymbol(ccl::g_stat_finds, &z, 8));
        CK(cudaMemcpyToSymbol(ccl::g_stat_hops, &z, 8));
        CK(cudaMemcpyToSymbol(ccl::g_stat_maxhops, &z, 8));
        ccl::k_boundary<TY, 8, 0><<<unsigned(bh + bv), 256>>>(g, bits, R, E, G, n_h, n_v);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpyFromSymbol(&u, ccl::g_stat_unions, 8));
        CK(cudaMemcpyFromSymbol(&st, ccl::g_stat_steps, 8));
        CK(cudaMemcpyFromSymbol(&nf, ccl::g_stat_finds, 8));
        CK(cudaMemcpyFromSymbol(&nh, ccl::g_stat_hops, 8));
        CK(cudaMemcpyFromSymbol(&mh, ccl::g_stat_maxhops, 8));
        printf("K2 stats: %llu union calls, %llu walk steps (%.2f per union)\n", u, st, double(st) / u);
        {
            unsigned long long ku, ks, kh;
            CK(cudaMemcpyToSymbol(ccl::g_stat_k1_unions, &z, 8));
            CK(cudaMemcpyToSymbol(ccl::g_stat_k1_steps, &z, 8));
            CK(cudaMemcpyToSymbol(ccl::g_stat_k1_hops, &z, 8));
            k1<<<grid1, ccl::k1_threads<TY>(), sm1>>>(img, g, bits, G, R, E, F, ntiles);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpyFromSymbol(&ku, ccl::g_stat_k1_unions, 8));
            CK(cudaMemcpyFromSymbol(&ks, ccl::g_stat_k1_steps, 8));
            CK(cudaMemcpyFromSymbol(&kh, ccl::g_stat_k1_hops, 8));
            printf("K1 stats: %llu unions, %.2f steps per union, %.2f find hops per union\n", ku, double(ks) / ku,
                   double(kh) / ku);
        }
        printf("K2 finds: %llu, %.2f hops avg, %llu max\n", nf, double(nh) / nf, mh);
    }
#endif
    // K3 (after K1 + K2), with stamps
    k1<<<grid1, ccl::k1_threads<TY>(), sm1>>>(img, g, bits, G, R, E, F, ntiles);
    ccl::k_boundary<TY, 8, 0><<<unsigned(bh + bv), 256>>>(g, bits, R, E, G, n_h, n_v);
    ccl::k_resolve<TY><<<std::min<unsigned>((ntiles + 7) / 8, 148 * 16), 256>>>(g, G, E, F, ntiles);
    auto k3 = ccl::k_link<TY, 8, true, true, true, 0>;
    auto k3s = ccl::k_link<TY, 8, true, true, true, 4>;
    const size_t sm3 = sizeof(ccl::LinkSmem<TY>);
    CUtensorMap tmap;
    {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        const cuuint64_t dims[3] = {32, cuuint64_t(W / 32), cuuint64_t(H)};
        const cuuint64_t strides[2] = {128, cuuint64_t(W) * 4};
        const cuuint32_t box[3] = {32, 32, 1}, es[3] = {1, 1, 1};
        if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            printf("tensor map encode failed\n");
    }
    CK(cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm3)));
    CK(cudaFuncSetAttribute(k3s, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm3)));
    for (int grid3 : {370, 390, 410, 428, 444}) {
        float us = timeit([&] { k3<<<grid3, ccl::kK3Threads, sm3>>>(g, bits, R, E, G, ccl::StripFinal{}, out, ntiles, tmap); }, flush, fb);
        printf("K3 grid %4d (%.2f tiles/block)     %8.1f us\n", grid3, double(ntiles) / grid3, us);
    }
    for (int per_sm : {3, 4, 5}) {
        const int grid3 = std::min<int>(ntiles, sms * per_sm);
        float us = timeit([&] { k3<<<grid3, ccl::kK3Threads, sm3>>>(g, bits, R, E, G, ccl::StripFinal{}, out, ntiles, tmap); }, flush, fb);
        printf("K3 x%d                              %8.1f us\n", per_sm, us);
    }
    {
        auto k3z = ccl::k_link<TY, 8, true, true, true, 1>;
        CK(cudaFuncSetAttribute(k3z, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm3)));
        float us = timeit([&] { k3z<<<std::min<int>(ntiles, sms * 3), ccl::kK3Threads, sm3>>>(g, bits, R, E, G, ccl::StripFinal{}, out, ntiles, tmap); }, flush, fb);
        printf("K3 x3, no expansion (stale rowbuf)  %8.1f us\n", us);
    }
    unsigned long long* st3;
    CK(cudaMalloc(&st3, size_t(ntiles) * 8 * 8));
    CK(cudaMemcpyToSymbol(ccl::g_k3_stamps, &st3, sizeof(st3)));
    float us3 = timeit([&] { k3s<<<std::min<int>(ntiles, sms * 4), ccl::kK3Threads, sm3>>>(g, bits, R, E, G, ccl::StripFinal{}, out, ntiles, tmap); }, flush, fb);
    printf("K3 + stamps x4                     %8.1f us\n", us3);
    CK(cudaMemcpy(hs.data(), st3, hs.size() * 8, cudaMemcpyDeviceToHost));
    const char* n3[3] = {"row runs", "label table", "expand+write"};
    double a3[3] = {0}, t3 = 0;
    for (unsigned t = 0; t < ntiles; ++t)
        for (int k = 0; k < 3; ++k) a3[k] += double(hs[t * 8 + k + 1] - hs[t * 8 + k]);
    for (int k = 0; k < 3; ++k) t3 += a3[k];
    for (int k = 0; k < 3; ++k) printf("  %-18s %8.0f  (%4.1f%%)\n", n3[k], a3[k] / ntiles, 100 * a3[k] / t3);
    return 0;
}
