// volume.cu — row a1: density grid -> device sampler layout.
//
// Every layout carries the 1-voxel zero apron of the canonical sampler
// (C1: padded index 0 and n+1 are vacuum), so the march kernel
// never bounds-checks a corner.  One thread per output element: the writes
// are fully coalesced, the gathers from the x-fastest raw grid are
// sector-coalesced along x.  HBM-bound: bytes = raw read + layout write.
#include <cstdlib>

#include <cuda_fp16.h>

#include "nsl_internal.cuh"

namespace nsl {

size_t layout_elems(int layout, int nx, int ny, int nz) {
    switch (layout) {
        case kLinearF32: return (size_t)(nx + 2) * (ny + 2) * (nz + 2);
        case kQuadF32: return (size_t)(nx + 1) * (ny + 1) * (nz + 2);
        case kCornerF16: return (size_t)(nx + 1) * (ny + 1) * (nz + 1);
    }
    return 0;
}

size_t layout_elem_bytes(int layout) {
    switch (layout) {
        case kLinearF32: return 4;
        case kQuadF32: return 16;
        case kCornerF16: return 16;
    }
    return 0;
}

namespace {

struct Raw {
    const float* __restrict__ v;
    int nx, ny, nz;
    // padded-index read: 0 outside [1, n]
    __device__ __forceinline__ float at(int i, int j, int k) const {
        if (i < 1 || j < 1 || k < 1 || i > nx || j > ny || k > nz) return 0.0f;
        return __ldg(v + ((size_t)(k - 1) * ny + (j - 1)) * nx + (i - 1));
    }
};

__device__ __forceinline__ void check(float x, unsigned long long* invalid) {
    if (!(x >= 0.0f) || isinf(x)) atomicAdd(invalid, 1ull);
}

__global__ void layout_linear_kernel(Raw r, float* __restrict__ out, unsigned long long* invalid, size_t total) {
    const int px = r.nx + 2, py = r.ny + 2;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        int i = (int)(e % px);
        size_t rest = e / px;
        int j = (int)(rest % py), k = (int)(rest / py);
        float x = r.at(i, j, k);
        if (i >= 1 && j >= 1 && k >= 1 && i <= r.nx && j <= r.ny && k <= r.nz) check(x, invalid);
        out[e] = x;
    }
}

__global__ void layout_quad_kernel(Raw r, float4* __restrict__ out, unsigned long long* invalid, size_t total) {
    const int qx = r.nx + 1, qy = r.ny + 1;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        int i = (int)(e % qx);
        size_t rest = e / qx;
        int j = (int)(rest % qy), k = (int)(rest / qy);
        // (c000, c100 - c000, c010, c110 - c010): the x-lerps of the march become one
        // FMA each, fma(fx, c100 - c000, c000), with the difference rounded exactly as
        // the kernel's own lerp would round it (bit-identical to the LINEAR layout)
        const float c000 = r.at(i, j, k), c100 = r.at(i + 1, j, k);
        const float c010 = r.at(i, j + 1, k), c110 = r.at(i + 1, j + 1, k);
        if (i >= 1 && j >= 1 && k >= 1 && k <= r.nz) check(c000, invalid);
        out[e] = make_float4(c000, __fsub_rn(c100, c000), c010, __fsub_rn(c110, c010));
    }
}

__global__ void layout_corner_f16_kernel(Raw r, uint4* __restrict__ out, unsigned long long* invalid, size_t total) {
    const int qx = r.nx + 1, qy = r.ny + 1;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        int i = (int)(e % qx);
        size_t rest = e / qx;
        int j = (int)(rest % qy), k = (int)(rest / qy);
        float c[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) c[b] = r.at(i + (b & 1), j + ((b >> 1) & 1), k + (b >> 2));
        if (i >= 1 && j >= 1 && k >= 1) check(c[0], invalid);
        __half2 h0 = __floats2half2_rn(c[0], c[1]), h1 = __floats2half2_rn(c[2], c[3]);
        __half2 h2 = __floats2half2_rn(c[4], c[5]), h3 = __floats2half2_rn(c[6], c[7]);
        uint4 u;
        u.x = *reinterpret_cast<unsigned*>(&h0);
        u.y = *reinterpret_cast<unsigned*>(&h1);
        u.z = *reinterpret_cast<unsigned*>(&h2);
        u.w = *reinterpret_cast<unsigned*>(&h3);
        out[e] = u;
    }
}

// One thread per occupancy block: the block is non-empty iff some padded
// voxel in [b*B, b*B + B]^3 (the corners of its cells) is nonzero.
__global__ void occupancy_kernel(Raw r, uint32_t* __restrict__ mask, OccGeom g, int32_t* __restrict__ aabb) {
    const int B = 1 << g.shift;
    const int total = g.nbx * g.nby * g.nbz;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < total; b += gridDim.x * blockDim.x) {
        const int bx = b % g.nbx, by = (b / g.nbx) % g.nby, bz = b / (g.nbx * g.nby);
        const int x0 = max(bx * B, 1), x1 = min(bx * B + B, r.nx);
        const int y0 = max(by * B, 1), y1 = min(by * B + B, r.ny);
        const int z0 = max(bz * B, 1), z1 = min(bz * B + B, r.nz);
        bool any = false;
        for (int k = z0; k <= z1 && !any; ++k)
            for (int j = y0; j <= y1 && !any; ++j)
                for (int i = x0; i <= x1; ++i)
                    if (r.at(i, j, k) != 0.0f) {
                        any = true;
                        break;
                    }
        if (any) {
            atomicOr(mask + (b >> 5), 1u << (b & 31));
            int32_t* smin = reinterpret_cast<int32_t*>(mask + g.words);
            int32_t* smax = smin + 2 * g.nbz;
            atomicMin(smin + 2 * bz, bx);
            atomicMin(smin + 2 * bz + 1, by);
            atomicMax(smax + 2 * bz, bx);
            atomicMax(smax + 2 * bz + 1, by);
            atomicMin(aabb + 0, bx);
            atomicMin(aabb + 1, by);
            atomicMin(aabb + 2, bz);
            atomicMax(aabb + 3, bx);
            atomicMax(aabb + 4, by);
            atomicMax(aabb + 5, bz);
        }
    }
}

}  // namespace

// Occupancy block size: the smallest 2^shift (shift >= 1) whose bitmask fits
// the per-CTA shared-memory budget (default 16 KB; NSL_OCC_BUDGET / NSL_OCC_SHIFT
// override for experiments).
OccGeom occ_geom(int nx, int ny, int nz) {
    long budget = 16 * 1024;   // ~33 blocks per axis; measured best on C2 (profiles/r1_sweep.txt)
    if (const char* e = getenv("NSL_OCC_BUDGET")) budget = atol(e);
    if (budget > 16 * 1024) budget = 16 * 1024;   // <= 2^17 blocks: the march's fp32 block index stays exact
    int forced = 0;
    if (const char* e = getenv("NSL_OCC_SHIFT")) forced = atoi(e);
    OccGeom g{};
    for (int s = forced > 0 ? forced : 1; s <= 10; ++s) {
        const int B = 1 << s;
        g.shift = s;
        g.nbx = (nx + 1 + B - 1) / B;
        g.nby = (ny + 1 + B - 1) / B;
        g.nbz = (nz + 1 + B - 1) / B;
        const long bits = (long)g.nbx * g.nby * g.nbz;
        g.words = (int)(((bits + 31) / 32 + 3) / 4 * 4);
        g.words_total = g.words + 4 * g.nbz;
        if ((forced > 0 && s >= forced) || (long)g.words * 4 <= budget) {
            if ((long)g.words * 4 <= 16 * 1024 && g.nbz <= 1024) break;
        }
    }
    return g;
}

cudaError_t launch_occupancy(const float* raw, const VolDesc& v, uint32_t* mask, int32_t* aabb, cudaStream_t s) {
    Raw r{raw, v.nx, v.ny, v.nz};
    cudaError_t e = cudaMemsetAsync(mask, 0, (size_t)v.og.words * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(mask + v.og.words, 0x7f, (size_t)v.og.nbz * 8, s);                 // slab min
    if (e == cudaSuccess) e = cudaMemsetAsync(mask + v.og.words + 2 * v.og.nbz, 0xff, (size_t)v.og.nbz * 8, s);  // slab max
    if (e == cudaSuccess) e = cudaMemsetAsync(aabb, 0x7f, 3 * sizeof(int32_t), s);      // bmin = 0x7f7f7f7f
    if (e == cudaSuccess) e = cudaMemsetAsync(aabb + 3, 0xff, 3 * sizeof(int32_t), s);  // bmax = -1
    if (e != cudaSuccess) return e;
    const int total = v.og.nbx * v.og.nby * v.og.nbz;
    occupancy_kernel<<<(total + 127) / 128, 128, 0, s>>>(r, mask, v.og, aabb);
    return cudaGetLastError();
}

cudaError_t launch_layout(const float* raw, const VolDesc& v, void* storage, unsigned long long* invalid,
                          cudaStream_t s) {
    Raw r{raw, v.nx, v.ny, v.nz};
    size_t total = layout_elems(v.layout, v.nx, v.ny, v.nz);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t want = (total + 255) / 256;
    unsigned blocks = (unsigned)(want < (size_t)sms * 16 ? want : (size_t)sms * 16);
    if (blocks == 0) blocks = 1;
    switch (v.layout) {
        case kLinearF32:
            layout_linear_kernel<<<blocks, 256, 0, s>>>(r, static_cast<float*>(storage), invalid, total);
            break;
        case kQuadF32:
            layout_quad_kernel<<<blocks, 256, 0, s>>>(r, static_cast<float4*>(storage), invalid, total);
            break;
        case kCornerF16:
            layout_corner_f16_kernel<<<blocks, 256, 0, s>>>(r, static_cast<uint4*>(storage), invalid, total);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace nsl
