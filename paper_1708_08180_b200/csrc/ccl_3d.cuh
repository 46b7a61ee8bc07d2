// ccl_3d.cuh -- 3D volumes ("2D/3D grid"):
// the same three phases over bricks.  Voxel (x,y,z) of a D x H x W volume has
// raster index (z*H + y)*W + x; foreground = nonzero; 6- or 26-connectivity;
// output 0 or 1 + the component's minimum raster index (the 2D convention).
//  local merge  one 32x4x4 brick per block: voxel-level min-root union-find
//               in shared memory over the in-brick backward neighbours, each
//               voxel's local root converted to its global index -> G;
//  boundary     every voxel with a backward neighbour in another brick unions
//               the two local roots in global memory (min-root, path
//               splitting);
//  link         every voxel -> 1 + root (k_link_flat of ccl_baselines.cuh).
// A pixel-level design (as the paper's own kernels): 3D is an adjacent row
// of the scope table, not the 2D hot path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ccl_baselines.cuh"

namespace ccl {
namespace vol {

constexpr int kX = 32, kY = 4, kZ = 4;  // brick = block (512 threads)

// the 13 backward neighbours (dz < 0, or dz == 0 and dy < 0, or dz == dy == 0
// and dx < 0); the first 3 are the 6-connectivity faces
__constant__ int8_t kNb[13][3] = {{-1, 0, 0}, {0, -1, 0}, {0, 0, -1},  // (dx, dy, dz)
                                  {-1, -1, 0}, {1, -1, 0},
                                  {-1, 0, -1}, {1, 0, -1}, {0, -1, -1}, {0, 1, -1},
                                  {-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {1, 1, -1}};

template <int CONN>
__global__ void __launch_bounds__(kX * kY * kZ) k_vol_local(const uint8_t* __restrict__ v, int D, int H, int W,
                                                            long long nvox, int bz_per_img,
                                                            int32_t* __restrict__ G) {
    __shared__ int32_t P[kX * kY * kZ];
    __shared__ uint8_t F[kX * kY * kZ];
    const int b = blockIdx.z / bz_per_img, bz = blockIdx.z % bz_per_img;
    const uint8_t* vb = v + size_t(b) * size_t(nvox);
    int32_t* Gb = G + size_t(b) * size_t(nvox);
    const int lx = threadIdx.x, ly = threadIdx.y, lz = threadIdx.z;
    const int t = (lz * kY + ly) * kX + lx;
    const int x = blockIdx.x * kX + lx, y = blockIdx.y * kY + ly, z = bz * kZ + lz;
    const bool in = x < W && y < H && z < D;
    const size_t p = (size_t(z) * H + y) * W + x;
    const bool f = in && vb[p] != 0;
    P[t] = t;
    F[t] = f;
    __syncthreads();
    if (f) {
        constexpr int NB = CONN == 6 ? 3 : 13;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const int xx = lx + kNb[k][0], yy = ly + kNb[k][1], zz = lz + kNb[k][2];
            if (xx < 0 || xx >= kX || yy < 0 || yy >= kY || zz < 0) continue;  // other brick: boundary phase
            const int t2 = (zz * kY + yy) * kX + xx;
            if (F[t2]) base::union_min(P, t, t2);
        }
    }
    __syncthreads();
    if (in) {
        int val = -1;
        if (f) {
            const int r = base::find_root(P, t);
            const int rx = blockIdx.x * kX + r % kX, ry = blockIdx.y * kY + (r / kX) % kY, rz = bz * kZ + r / (kX * kY);
            val = int((size_t(rz) * H + ry) * W + rx);
        }
        Gb[p] = val;
    }
}

// one thread per voxel; interior voxels (no backward neighbour outside the
// brick) return at once
template <int CONN>
__global__ void k_vol_boundary(const uint8_t* __restrict__ v, int D, int H, int W, long long nvox,
                               int32_t* __restrict__ G) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (i >= nvox) return;
    const int x = int(i % W), y = int((i / W) % H), z = int(i / ((long long)W * H));
    const int lx = x % kX, ly = y % kY, lz = z % kZ;
    const bool edge = lx == 0 || lz == 0 || ly == 0 || (CONN == 26 && (lx == kX - 1 || ly == kY - 1));
    if (!edge) return;
    const uint8_t* vb = v + size_t(b) * size_t(nvox);
    if (vb[i] == 0) return;
    int32_t* Gb = G + size_t(b) * size_t(nvox);
    constexpr int NB = CONN == 6 ? 3 : 13;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const int dx = kNb[k][0], dy = kNb[k][1], dz = kNb[k][2];
        const int xx = x + dx, yy = y + dy, zz = z + dz;
        if (xx < 0 || xx >= W || yy < 0 || yy >= H || zz < 0) continue;
        const int lxx = lx + dx, lyy = ly + dy, lzz = lz + dz;
        if (lxx >= 0 && lxx < kX && lyy >= 0 && lyy < kY && lzz >= 0) continue;  // same brick: local phase
        const size_t q = (size_t(zz) * H + yy) * W + xx;
        if (vb[q] != 0) base::union_min(Gb, Gb[i], Gb[q]);
    }
}

}  // namespace vol
}  // namespace ccl
