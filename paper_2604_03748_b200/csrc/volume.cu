// volume.cu — row a1: density grid -> device sampler layout.
//
// Every layout carries the 1-voxel zero apron of the canonical sampler
// (C1: padded index 0 and n+1 are vacuum), so the march kernel
// never bounds-checks a corner.  One thread per output element: the writes
// are fully coalesced, the gathers from the x-fastest raw grid are
// sector-coalesced along x.  HBM-bound: bytes = raw read + layout write.
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include "nsl_internal.cuh"

namespace nsl {

size_t layout_elems(int layout, int nx, int ny, int nz) {
    switch (layout) {
        case kLinearF32: return (size_t)(nx + 2) * (ny + 2) * (nz + 2);
        case kQuadF32: return (size_t)(nx + 1) * (ny + 1) * (nz + 2);
        case kCornerF16: return (size_t)(nx + 1) * (ny + 1) * (nz + 1);
        case kOctF32: return (size_t)(nx + 1) * (ny + 1) * (nz + 1);
        case kBrickOctF32: return (size_t)((nx + 4) / 4) * ((ny + 4) / 4) * ((nz + 4) / 4) * 64;
        case kMortonOctF32: return (size_t)((nx + 8) / 8) * ((ny + 8) / 8) * ((nz + 8) / 8) * 512;
        case kTex3dF32: return 0;      // the body lives in the library-owned cudaArray
    }
    return 0;
}

size_t layout_elem_bytes(int layout) {
    switch (layout) {
        case kLinearF32: return 4;
        case kQuadF32: return 16;
        case kCornerF16: return 16;
        case kOctF32: return 32;
        case kBrickOctF32: return 32;
        case kMortonOctF32: return 32;
        case kTex3dF32: return 16;
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

// ---------------------------------------------------------------- layout role (one CTA = 256
// consecutive elements of one padded z-plane, i fastest; 32-bit index arithmetic)
__device__ __forceinline__ void layout_linear_cta(const Raw& r, float* __restrict__ out, int pb, int kb, int kstep) {
    const int px = r.nx + 2, py = r.ny + 2, plane = px * py;
    const int e2 = pb * 256 + threadIdx.x;
    if (e2 >= plane) return;
    const int i = e2 % px, j = e2 / px;
    for (int k = kb; k < r.nz + 2; k += kstep) out[(size_t)k * plane + e2] = r.at(i, j, k);
}

// QUAD: each thread writes kQuadPlanes planes (k, k + kstep, ...) with all raw loads issued
// before the stores (more bytes in flight per thread; HBM-bound).
constexpr int kQuadPlanes = 2;
__device__ __forceinline__ void layout_quad_cta(const Raw& r, float4* __restrict__ out, int pb, int kb, int kstep) {
    const int qx = r.nx + 1, qy = r.ny + 1, plane = qx * qy;
    const int e2 = pb * 256 + threadIdx.x;
    if (e2 >= plane) return;
    const int i = e2 % qx, j = e2 / qx;
    for (; kb < r.nz + 2; kb += kstep * kQuadPlanes) {
        float c[kQuadPlanes][4];
#pragma unroll
        for (int t = 0; t < kQuadPlanes; ++t) {
            const int k = kb + t * kstep;
            c[t][0] = r.at(i, j, k);
            c[t][1] = r.at(i + 1, j, k);
            c[t][2] = r.at(i, j + 1, k);
            c[t][3] = r.at(i + 1, j + 1, k);
        }
#pragma unroll
        for (int t = 0; t < kQuadPlanes; ++t) {
            const int k = kb + t * kstep;
            if (k >= r.nz + 2) break;
            // (c000, c100 - c000, c010, c110 - c010): the x-lerps of the march become one
            // FMA each, fma(fx, c100 - c000, c000), with the difference rounded exactly as
            // the kernel's own lerp would round it (bit-identical to the LINEAR layout)
            out[(size_t)k * plane + e2] =
                make_float4(c[t][0], __fsub_rn(c[t][1], c[t][0]), c[t][2], __fsub_rn(c[t][3], c[t][2]));
        }
    }
}

__device__ __forceinline__ void layout_corner_f16_cta(const Raw& r, uint4* __restrict__ out, int pb, int kb,
                                                      int kstep) {
    const int qx = r.nx + 1, qy = r.ny + 1, plane = qx * qy;
    const int e2 = pb * 256 + threadIdx.x;
    if (e2 >= plane) return;
    const int i = e2 % qx, j = e2 / qx;
    for (int k = kb; k < r.nz + 1; k += kstep) {
        float c[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) c[b] = r.at(i + (b & 1), j + ((b >> 1) & 1), k + (b >> 2));
        __half2 h0 = __floats2half2_rn(c[0], c[1]), h1 = __floats2half2_rn(c[2], c[3]);
        __half2 h2 = __floats2half2_rn(c[4], c[5]), h3 = __floats2half2_rn(c[6], c[7]);
        uint4 u;
        u.x = *reinterpret_cast<unsigned*>(&h0);
        u.y = *reinterpret_cast<unsigned*>(&h1);
        u.z = *reinterpret_cast<unsigned*>(&h2);
        u.w = *reinterpret_cast<unsigned*>(&h3);
        out[(size_t)k * plane + e2] = u;
    }
}

// OCT: the QUAD float4 of planes k and k+1 of cell (i, j, k) in one 32-B element (k <= nz).
// Each thread walks a run of kOctRun consecutive planes carrying plane k+1's quad into the
// next element (4 raw loads per element instead of 8) and writes each element with one
// 256-bit store.
#ifndef NSL_OCT_RUN
#define NSL_OCT_RUN 8
#endif
#ifndef NSL_OCT_UNROLL
#define NSL_OCT_UNROLL 4   // measured on C4 (60 x 256^3 builds): 8.29 -> 7.98 ms
#endif
constexpr int kOctRun = NSL_OCT_RUN, kOctUnroll = NSL_OCT_UNROLL;
__device__ __forceinline__ void st256(float* p, const float (&c)[8]) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(c[0]), "f"(c[1]),
                 "f"(c[2]), "f"(c[3]), "f"(c[4]), "f"(c[5]), "f"(c[6]), "f"(c[7])
                 : "memory");
}
__device__ __forceinline__ void layout_oct_cta(const Raw& r, float* __restrict__ out, int pb, int kb, int kstep) {
    const int qx = r.nx + 1, qy = r.ny + 1, plane = qx * qy;
    const int e2 = pb * 256 + threadIdx.x;
    if (e2 >= plane) return;
    const int i = e2 % qx, j = e2 / qx;
    // the x/y apron tests and row offsets are fixed per thread: padded corner a is real iff
    // 1 <= a <= n; raw offset of padded (a, b, c) = ((c - 1) ny + b - 1) nx + a - 1
    const bool x0 = i >= 1, x1 = i < r.nx, y0 = j >= 1, y1 = j < r.ny;
    const bool c00 = x0 && y0, c10 = x1 && y0, c01 = x0 && y1, c11 = x1 && y1;
    const int64_t zs = (int64_t)r.nx * r.ny, o00 = (int64_t)(j - 1) * r.nx + (i - 1);
    auto quad = [&](int c, float (&d)[4]) {           // the 2x2 x/y corners of padded plane c
        const bool pc = c >= 1 && c <= r.nz;
        const float* b = r.v + (o00 + (int64_t)(c - 1) * zs);
        d[0] = pc && c00 ? __ldg(b) : 0.0f;
        d[1] = pc && c10 ? __ldg(b + 1) : 0.0f;
        d[2] = pc && c01 ? __ldg(b + r.nx) : 0.0f;
        d[3] = pc && c11 ? __ldg(b + r.nx + 1) : 0.0f;
    };
    for (int k0 = kb * kOctRun; k0 < r.nz + 1; k0 += kstep * kOctRun) {
        const int k1 = min(k0 + kOctRun, r.nz + 1);
        float q[4];
        quad(k0, q);
#pragma unroll kOctUnroll
        for (int k = k0; k < k1; ++k) {
            float n[4];
            quad(k + 1, n);
            // (c000, c100 - c000, c010, c110 - c010 | the same for plane k+1): the differences are
            // rounded exactly as the sampler's lerp rounds them (bit-identical to LINEAR)
            const float c[8] = {q[0], __fsub_rn(q[1], q[0]), q[2], __fsub_rn(q[3], q[2]),
                                n[0], __fsub_rn(n[1], n[0]), n[2], __fsub_rn(n[3], n[2])};
            st256(out + 8 * ((size_t)k * plane + e2), c);
#pragma unroll
            for (int t = 0; t < 4; ++t) q[t] = n[t];
        }
    }
}

// BRICK_OCT: element e = brick * 64 + (i & 3) + 4 (j & 3) + 16 (k & 3), brick = ((k >> 2) nby_b +
// (j >> 2)) nbx_b + (i >> 2); one thread per element (coalesced 256-bit stores), cells beyond
// (n_x, n_y, n_z) in the last bricks hold zeros (never sampled).
__device__ __forceinline__ void layout_brick_oct_cta(const Raw& r, float* __restrict__ out, int pb) {
    const int nbx = (r.nx + 4) / 4, nby = (r.ny + 4) / 4, nbz = (r.nz + 4) / 4;
    const int64_t e = (int64_t)pb * 256 + threadIdx.x;
    if (e >= (int64_t)nbx * nby * nbz * 64) return;
    const int off = (int)(e & 63);
    const int64_t b = e >> 6;
    const int bx = (int)(b % nbx), by = (int)((b / nbx) % nby), bz = (int)(b / ((int64_t)nbx * nby));
    const int i = bx * 4 + (off & 3), j = by * 4 + ((off >> 2) & 3), k = bz * 4 + (off >> 4);
    float c[8];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const float c0 = r.at(i, j, k + t), c1 = r.at(i + 1, j, k + t);
        const float c2 = r.at(i, j + 1, k + t), c3 = r.at(i + 1, j + 1, k + t);
        c[4 * t + 0] = c0;
        c[4 * t + 1] = __fsub_rn(c1, c0);
        c[4 * t + 2] = c2;
        c[4 * t + 3] = __fsub_rn(c3, c2);
    }
    st256(out + 8 * e, c);
}

// MORTON_OCT: element e = tile * 512 + morton(i & 7, j & 7, k & 7) (bit b of the x offset at bit
// 3b, y at 3b + 1, z at 3b + 2), tile = ((k >> 3) nty + (j >> 3)) ntx + (i >> 3); one thread per
// element, cells beyond (n_x, n_y, n_z) in the last tiles hold zeros (never sampled).
__device__ __forceinline__ void layout_morton_oct_cta(const Raw& r, float* __restrict__ out, int pb) {
    const int ntx = (r.nx + 8) / 8, nty = (r.ny + 8) / 8, ntz = (r.nz + 8) / 8;
    const int64_t e = (int64_t)pb * 256 + threadIdx.x;
    if (e >= (int64_t)ntx * nty * ntz * 512) return;
    const int m = (int)(e & 511);
    const int64_t t = e >> 9;
    const int tx = (int)(t % ntx), ty = (int)((t / ntx) % nty), tz = (int)(t / ((int64_t)ntx * nty));
    const int ox = (m & 1) | ((m >> 2) & 2) | ((m >> 4) & 4);
    const int oy = ((m >> 1) & 1) | ((m >> 3) & 2) | ((m >> 5) & 4);
    const int oz = ((m >> 2) & 1) | ((m >> 4) & 2) | ((m >> 6) & 4);
    const int i = tx * 8 + ox, j = ty * 8 + oy, k = tz * 8 + oz;
    float c[8];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const float c0 = r.at(i, j, k + q), c1 = r.at(i + 1, j, k + q);
        const float c2 = r.at(i, j + 1, k + q), c3 = r.at(i + 1, j + 1, k + q);
        c[4 * q + 0] = c0;
        c[4 * q + 1] = __fsub_rn(c1, c0);
        c[4 * q + 2] = c2;
        c[4 * q + 3] = __fsub_rn(c3, c2);
    }
    st256(out + 8 * e, c);
}

// TEX3D: the QUAD float4 of padded cell (i, j, k) written through the array's surface object
// (texel (i, j, k); x in bytes), one thread per cell of a z-plane, planes k = kb, kb + kstep, ...
__device__ __forceinline__ void layout_tex3d_cta(const Raw& r, cudaSurfaceObject_t surf, int pb, int kb, int kstep) {
    const int qx = r.nx + 1, qy = r.ny + 1, plane = qx * qy;
    const int e2 = pb * 256 + threadIdx.x;
    if (e2 >= plane) return;
    const int i = e2 % qx, j = e2 / qx;
    for (int k = kb; k < r.nz + 2; k += kstep) {
        const float c0 = r.at(i, j, k), c1 = r.at(i + 1, j, k), c2 = r.at(i, j + 1, k), c3 = r.at(i + 1, j + 1, k);
        surf3Dwrite(make_float4(c0, __fsub_rn(c1, c0), c2, __fsub_rn(c3, c2)), surf, i * (int)sizeof(float4), j, k);
    }
}

// ---------------------------------------------------------------- occupancy role
// Block (bx, by, bz) is non-empty iff some padded voxel in [b*B, b*B + B]^3 (the corners of
// its cells) is nonzero; voxel i is a corner of the cells i-1 and i, i.e. of the blocks
// (i-1)>>s and i>>s.  One CTA per block row (by, bz): its warps stream the (B+1)^2 raw
// x-rows of the row (coalesced, kOccChunks x 32 voxels in flight per warp, one ballot per
// 32), OR the x-block flags into shared memory and write them, with the row's x extent and
// its count of invalid voxels (the rows j in [by B, by B + B), k in [bz B, bz B + B) only, so
// each voxel is counted once), to the row's scratch record: plain stores, no atomics, no
// initialisation.  occ_finalize_kernel assembles mask, slab boxes, AABB and the count.
constexpr int kOccChunks = 4;   // 32-voxel chunks per row loaded at once
constexpr int kOccRows = 2;     // rows per warp loaded at once
__device__ __forceinline__ void occupancy_cta(const Raw& r, const OccGeom& g, uint32_t* __restrict__ scratch,
                                              int row_id, uint32_t* xflag, int* red) {
    const int s = g.shift, B = 1 << s;
    const int by = row_id % g.nby, bz = row_id / g.nby;
    for (int w = threadIdx.x; w < g.rowwords; w += blockDim.x) xflag[w] = 0u;
    if (threadIdx.x == 0) {
        red[0] = 0x7fffffff;
        red[1] = -1;
        red[2] = 0;
    }
    __syncthreads();
    const int j0 = max(by * B, 1), j1 = min(by * B + B, r.ny);
    const int k0 = max(bz * B, 1), k1 = min(bz * B + B, r.nz);
    const int nj = j1 - j0 + 1, nrows = nj > 0 && k1 >= k0 ? nj * (k1 - k0 + 1) : 0;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = blockDim.x / 32;
    int bad = 0;
    for (int row0 = warp; row0 < nrows; row0 += nwarps * kOccRows) {
        // kOccRows rows x kOccChunks chunks of 32 voxels: all loads in flight together
        float x[kOccRows][kOccChunks];
#pragma unroll
        for (int q = 0; q < kOccRows; ++q) {
            const int row = row0 + q * nwarps;
            const int j = j0 + row % nj, k = k0 + row / nj;
            const float* src = r.v + ((size_t)(k - 1) * r.ny + (j - 1)) * r.nx;
#pragma unroll
            for (int t = 0; t < kOccChunks; ++t) {
                const int i = 1 + 32 * t + lane;
                x[q][t] = row < nrows && i <= r.nx ? __ldg(src + (i - 1)) : 0.0f;
            }
        }
#pragma unroll
        for (int q = 0; q < kOccRows; ++q) {
            const int row = row0 + q * nwarps;
            if (row >= nrows) break;
            const int j = j0 + row % nj, k = k0 + row / nj;
            const bool counted = j < by * B + B && k < bz * B + B;
            const float* src = r.v + ((size_t)(k - 1) * r.ny + (j - 1)) * r.nx;
            for (int g0 = 1; g0 <= r.nx; g0 += 32 * kOccChunks) {
                float xv[kOccChunks];
#pragma unroll
                for (int t = 0; t < kOccChunks; ++t) {
                    const int i = g0 + 32 * t + lane;
                    xv[t] = g0 == 1 ? x[q][t] : (i <= r.nx ? __ldg(src + (i - 1)) : 0.0f);
                }
#pragma unroll
                for (int t = 0; t < kOccChunks; ++t) {
                    const int c0 = g0 + 32 * t, i = c0 + lane;
                    bad += counted && i <= r.nx && (!(xv[t] >= 0.0f) || isinf(xv[t]));
                    const bool nz = xv[t] != 0.0f;
                    if (!__any_sync(0xffffffffu, nz)) continue;
                    // x-blocks of this chunk lie in bit words wa, wa+1 (32 voxels span <= 32/B + 2 blocks)
                    const int wa = ((c0 - 1) >> s) >> 5;
                    unsigned b0 = 0u, b1 = 0u;
                    if (nz) {
                        const int xa = (i - 1) >> s, xb = i >> s;
                        (xa >> 5 == wa ? b0 : b1) |= 1u << (xa & 31);
                        if (xb < g.nbx) (xb >> 5 == wa ? b0 : b1) |= 1u << (xb & 31);
                    }
                    b0 = __reduce_or_sync(0xffffffffu, b0);
                    b1 = __reduce_or_sync(0xffffffffu, b1);
                    if (lane == 0) {
                        if (b0) atomicOr(xflag + wa, b0);
                        if (b1) atomicOr(xflag + wa + 1, b1);
                    }
                }
            }
        }
    }
    bad = __reduce_add_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicAdd(red + 2, bad);
    __syncthreads();
    for (int bx = threadIdx.x; bx < g.nbx; bx += blockDim.x)
        if (xflag[bx >> 5] >> (bx & 31) & 1u) {
            atomicMin(red + 0, bx);
            atomicMax(red + 1, bx);
        }
    uint32_t* flags = scratch + (size_t)row_id * g.rowwords;
    for (int w = threadIdx.x; w < g.rowwords; w += blockDim.x) flags[w] = xflag[w];
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t* info = reinterpret_cast<int32_t*>(scratch + g.info_off) + 4 * row_id;
        info[0] = red[0];
        info[1] = red[1];
        info[2] = red[2];
    }
}

// Horizontal fusion of the two independent passes over the raw grid: CTAs [0, rows) are
// occupancy rows, the rest write the sampler layout.  Triggers its dependent (the
// PDL-launched occ_finalize_kernel) at once so that launch overlaps this grid.
template <int LAYOUT>
__global__ void __launch_bounds__(256, 6) volume_build_kernel(Raw r, void* __restrict__ out, OccGeom g,
                                                              uint32_t* __restrict__ scratch, int plane_blocks,
                                                              int kstep, int occ_stride) {
    extern __shared__ uint32_t xflag[];
    __shared__ int red[3];
    pdl_trigger();
    // occupancy CTAs interleaved with the layout CTAs (every occ_stride-th of the first
    // rows*occ_stride) so that every wave mixes latency-bound scans with HBM streaming
    const int b = blockIdx.x;
    int lb;
    if (b < g.rows * occ_stride) {
        if (b % occ_stride == 0) {
            occupancy_cta(r, g, scratch, b / occ_stride, xflag, red);
            return;
        }
        lb = b - (b / occ_stride + 1);
    } else {
        lb = b - g.rows;
    }
    const int pb = lb % plane_blocks, kb = lb / plane_blocks;
    if (LAYOUT == kLinearF32) layout_linear_cta(r, static_cast<float*>(out), pb, kb, kstep);
    if (LAYOUT == kQuadF32) layout_quad_cta(r, static_cast<float4*>(out), pb, kb, kstep);
    if (LAYOUT == kCornerF16) layout_corner_f16_cta(r, static_cast<uint4*>(out), pb, kb, kstep);
    if (LAYOUT == kOctF32) layout_oct_cta(r, static_cast<float*>(out), pb, kb, kstep);
    if (LAYOUT == kBrickOctF32) layout_brick_oct_cta(r, static_cast<float*>(out), pb);
    if (LAYOUT == kMortonOctF32) layout_morton_oct_cta(r, static_cast<float*>(out), pb);
    if (LAYOUT == kTex3dF32)             // `out` carries the array's surface object
        layout_tex3d_cta(r, (cudaSurfaceObject_t)reinterpret_cast<uintptr_t>(out), pb, kb, kstep);
}

// The occupancy region [mask: words][slab_min: nbz x (bx, by)][slab_max: nbz x (bx, by)], the
// occupied-block AABB (bmin xyz, bmax xyz; bmin > bmax: empty) and the invalid-voxel count, from
// the rows' scratch records.  CTA 0 reduces the records (one thread per record, shared-memory
// min/max per slab; empty slab: min = 0x7f7f7f7f, max = -1); CTAs 1.. assemble the mask, one
// warp per 32-bit word, one lane per bit (a single gather each, then a ballot).
constexpr int kFinThreads = 1024;
__global__ void __launch_bounds__(kFinThreads) occ_finalize_kernel(OccGeom g, const uint32_t* __restrict__ scratch,
                                                                   uint32_t* __restrict__ mask,
                                                                   int32_t* __restrict__ aabb,
                                                                   unsigned long long* __restrict__ invalid) {
    // grid = 1 CTA when the mask was written by the build itself (oct_build_kernel)
    pdl_trigger();
    pdl_wait();
    const int32_t* info = reinterpret_cast<const int32_t*>(scratch + g.info_off);
    if (blockIdx.x > 0) {
        const long bits = (long)g.nbx * g.nby * g.nbz;
        const int w = (blockIdx.x - 1) * (kFinThreads / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
        if (w >= g.words) return;
        const long b = 32L * w + lane;
        bool bit = false;
        if (b < bits) {
            const int row = (int)(b / g.nbx), bx = (int)(b - (long)row * g.nbx);
            bit = __ldg(scratch + (size_t)row * g.rowwords + (bx >> 5)) >> (bx & 31) & 1u;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, bit);
        if (lane == 0) mask[w] = word;
        return;
    }
    // CTA 0: one warp per z slab reduces its rows' records (x extent, row occupied, invalid
    // voxels) with warp reductions into the slab box; the AABB from the slab boxes
    __shared__ int am[6];
    __shared__ unsigned long long nbad;
    if (threadIdx.x < 6) am[threadIdx.x] = threadIdx.x < 3 ? 0x7f7f7f7f : -1;
    if (threadIdx.x == 0) nbad = 0ull;
    __syncthreads();
    int32_t* smin = reinterpret_cast<int32_t*>(mask + g.words);
    int32_t* smax = smin + 2 * g.nbz;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long mybad = 0ull;
    for (int bz = warp; bz < g.nbz; bz += kFinThreads / 32) {
        int x0 = 0x7f7f7f7f, y0 = 0x7f7f7f7f, x1 = -1, y1 = -1;
        for (int by = lane; by < g.nby; by += 32) {
            const int4 rec = __ldg(reinterpret_cast<const int4*>(info) + bz * g.nby + by);
            mybad += (unsigned long long)rec.z;
            if (rec.y >= 0) {
                x0 = min(x0, rec.x);
                x1 = max(x1, rec.y);
                y0 = min(y0, by);
                y1 = max(y1, by);
            }
        }
        x0 = __reduce_min_sync(0xffffffffu, x0);
        y0 = __reduce_min_sync(0xffffffffu, y0);
        x1 = __reduce_max_sync(0xffffffffu, x1);
        y1 = __reduce_max_sync(0xffffffffu, y1);
        if (lane == 0) {
            smin[2 * bz] = x0;
            smin[2 * bz + 1] = y0;
            smax[2 * bz] = x1;
            smax[2 * bz + 1] = y1;
            if (x1 >= 0) {
                atomicMin(am + 0, x0);
                atomicMin(am + 1, y0);
                atomicMin(am + 2, bz);
                atomicMax(am + 3, x1);
                atomicMax(am + 4, y1);
                atomicMax(am + 5, bz);
            }
        }
    }
    if (mybad) atomicAdd(&nbad, mybad);
    __syncthreads();
    if (threadIdx.x < 6) aabb[threadIdx.x] = am[threadIdx.x];
    if (threadIdx.x == 0) *invalid = nbad;
}

// ---------------------------------------------------------------- OCT, staged and occupancy-gated
// (blocks of 4^3 or 8^3 cells).  The march reads an element only after its occupancy block's bit
// is set (sample(), sampler.cuh), and the bit is "some corner of some cell of the block is != 0",
// so the elements of empty blocks -- ~80 % of a plume's -- are never read and are not written:
// the build's 32 B/cell of writes drop ~5x.  One CTA = a 32 (x) x 8 (y) tile of cells, one block
// layer (B cells of z) per iteration: the layer's padded corner voxels, (32+1) x (8+1) x (B+1),
// are staged in shared memory by cp.async (zero-fill outside 1..n: the apron, no branches),
// then each thread tests its cell column's corners (the block bit: a warp ballot + a shared OR
// per block row), counts its own voxels that are negative / non-finite, and writes its B
// elements if its block is occupied.  The block bits go straight into the occupancy mask and the
// per-row x extents into the scratch records (the occupancy role's format) by atomics;
// occ_reset_kernel clears both first (the build waits for it before its first atomic) and
// occ_finalize_kernel's CTA 0 alone turns the records into slab boxes and the AABB.  The
// separate latency-bound occupancy scan (one CTA per block row) and the mask assembly
// disappear: the raw grid is read once, through shared memory (TMA).
// staged row: 40 voxels from raw x = i0 - 4 (a TMA box must start 16-B aligned in x): padded
// x = i0 + t at column t + kStX0
constexpr int kStTx = 32, kStTy = 8, kStRw = 40, kStX0 = 3;
__device__ __forceinline__ void cp_async4(uint32_t saddr, const float* src, bool real) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(saddr), "l"(src), "r"(real ? 4 : 0)
                 : "memory");
}

__global__ void __launch_bounds__(256) occ_reset_kernel(OccGeom g, uint32_t* __restrict__ mask,
                                                        uint32_t* __restrict__ scratch) {
    pdl_trigger();
    for (int t = blockIdx.x * 256 + threadIdx.x; t < g.words + g.rows; t += gridDim.x * 256) {
        if (t < g.words) mask[t] = 0u;
        else reinterpret_cast<int4*>(scratch + g.info_off)[t - g.words] = make_int4(0x7fffffff, -1, 0, 0);
    }
}

// TMA: the layer's (40, 9, B+1) raw box at raw (i0-4, j0-1, k0-1), one bulk-tensor copy issued by
// one thread; out-of-range voxels (the apron and beyond) arrive as zeros (OOB fill NONE).
__device__ __forceinline__ void tma_box3(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
}

template <int SHIFT, bool TMA>
__global__ void __launch_bounds__(256) oct_build_kernel(const __grid_constant__ CUtensorMap map, Raw r,
                                                        float* __restrict__ out, OccGeom g,
                                                        uint32_t* __restrict__ mask, uint32_t* __restrict__ scratch,
                                                        int tiles_x) {
    constexpr int B = 1 << SHIFT, NP = B + 1, RW = kStRw, RH = kStTy + 1, PL = RW * RH;
    __shared__ __align__(128) float brick[NP * PL];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t s_any[kStTy >> SHIFT > 0 ? kStTy >> SHIFT : 1];
    pdl_trigger();
    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
    const int i0 = (blockIdx.x % tiles_x) * kStTx, j0 = (blockIdx.x / tiles_x) * kStTy;
    const int i = i0 + lane, j = j0 + wy, qx = r.nx + 1, qy = r.ny + 1;
    const size_t plane = (size_t)qx * qy;
    const int nlayers = (r.nz + 1 + B - 1) >> SHIFT;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(brick);
    const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
    const uint32_t group = ((1u << B) - 1u) << (lane & ~(B - 1));
    const float* bp = brick + wy * RW + kStX0 + lane;
    if (TMA && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    bool waited = false;
    uint32_t phase = 0;
    for (int zb = blockIdx.y; zb < nlayers; zb += gridDim.y, phase ^= 1u) {
        const int k0 = zb << SHIFT;
        if (TMA) {
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // after the last layer's reads
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar),
                             "r"((uint32_t)(NP * PL * 4))
                             : "memory");
                tma_box3(sbase, &map, i0 - 4, j0 - 1, k0 - 1, sbar);
            }
        } else {                 // one staged row (c, y) per warp iteration: lanes 0-31 + lane 0's x = 32
            const bool xr = i >= 1 && i <= r.nx, xr32 = i0 + 32 <= r.nx;
            for (int row = wy; row < NP * RH; row += 8) {
                const int c = row / RH, y = row - c * RH, pk = k0 + c, pj = j0 + y;
                const bool rr = pj >= 1 && pj <= r.ny && pk >= 1 && pk <= r.nz;
                const float* src = r.v + (rr ? ((size_t)(pk - 1) * r.ny + (pj - 1)) * r.nx + (i0 - 1) : 0);
                const uint32_t dst = sbase + 4u * (row * RW + kStX0 + lane);
                cp_async4(dst, rr && xr ? src + lane : r.v, rr && xr);
                if (lane == 0) cp_async4(dst + 128u, rr && xr32 ? src + 32 : r.v, rr && xr32);
            }
        }
        if (threadIdx.x < (kStTy >> SHIFT > 0 ? kStTy >> SHIFT : 1)) s_any[threadIdx.x] = 0u;
        if (TMA) mbar_wait(sbar, phase);
        else asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        bool any = false;
        int bad = 0;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
            const float* p = bp + c * PL;
            any |= (p[0] != 0.0f) | (p[1] != 0.0f) | (p[RW] != 0.0f) | (p[RW + 1] != 0.0f);
            if (c < B) bad += !(p[0] >= 0.0f) || isinf(p[0]);     // own voxel (apron zeros: not bad)
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, any);
        if (lane == 0 && bal) atomicOr(s_any + (wy >> SHIFT), bal);
        bad = __reduce_add_sync(0xffffffffu, bad);
        __syncthreads();
        if (!waited) {                                             // occ_reset_kernel's writes
            pdl_wait();
            waited = true;
        }
        const bool occ = (s_any[wy >> SHIFT] & group) != 0;
        int* info = reinterpret_cast<int*>(scratch + g.info_off);
        if (occ && (wy & (B - 1)) == 0 && (lane & (B - 1)) == 0) {   // one thread per occupied block
            const int bx = i >> SHIFT, row = zb * g.nby + (j >> SHIFT), b = row * g.nbx + bx;
            atomicOr(mask + (b >> 5), 1u << (b & 31));
            atomicMin(info + 4 * row, bx);
            atomicMax(info + 4 * row + 1, bx);
        }
        if (lane == 0 && bad) atomicAdd(info + 4 * (zb * g.nby + (j >> SHIFT)) + 2, bad);
        if (occ && i < qx && j < qy) {
#pragma unroll
            for (int c = 0; c < B; ++c) {
                const int k = k0 + c;
                if (k > r.nz) break;
                const float* p = bp + c * PL;
                const float* q = p + PL;
                // (c000, c100 - c000, c010, c110 - c010 | plane k + 1): as layout_oct_cta
                const float e[8] = {p[0], __fsub_rn(p[1], p[0]), p[RW], __fsub_rn(p[RW + 1], p[RW]),
                                    q[0], __fsub_rn(q[1], q[0]), q[RW], __fsub_rn(q[RW + 1], q[RW])};
                st256(out + 8 * ((size_t)k * plane + (size_t)j * qx + i), e);
            }
        }
        __syncthreads();                                           // brick and s_any are reused
    }
}

}  // namespace

// Occupancy block size: the smallest 2^shift, shift >= 2 (4^3-cell blocks), whose bitmask fits
// a 64 KB budget (NSL_OCC_BUDGET / NSL_OCC_SHIFT override for experiments).  Measured with the
// per-tile ranges (round 2, step ms): 128^3 (C2) 4^3 blocks best (2^3: march -2 % but build
// +43 %); 256^3 (C3) 4^3 vs 8^3: march -5.2 %, step -5.0 %; C4 step -0.3 %; 512^3 (C5) 8^3 vs
// 16^3: march -5.3 % (4^3 would need a 268 KB mask).
OccGeom occ_geom(int nx, int ny, int nz) {
    constexpr long kMaxMask = 256 * 1024;   // hard cap (the march reads the mask through L1)
    long budget = 64 * 1024;
    if (const char* e = getenv("NSL_OCC_BUDGET")) budget = atol(e);
    if (budget > kMaxMask) budget = kMaxMask;
    int forced = 0;
    if (const char* e = getenv("NSL_OCC_SHIFT")) forced = atoi(e);
    OccGeom g{};
    for (int s = forced > 0 ? forced : 2; s <= 10; ++s) {
        const int B = 1 << s;
        g.shift = s;
        g.nbx = (nx + 1 + B - 1) / B;
        g.nby = (ny + 1 + B - 1) / B;
        g.nbz = (nz + 1 + B - 1) / B;
        const long bits = (long)g.nbx * g.nby * g.nbz;
        g.words = (int)(((bits + 31) / 32 + 3) / 4 * 4);
        g.words_total = g.words + 4 * g.nbz;
        g.rowwords = (g.nbx + 31) / 32;
        g.rows = g.nby * g.nbz;
        g.info_off = (g.rows * g.rowwords + 3) / 4 * 4;
        g.scratch_words = g.info_off + 4 * g.rows;
        if ((forced > 0 && s >= forced) || (long)g.words * 4 <= budget) {
            if ((long)g.words * 4 <= kMaxMask && g.nbz <= 1024) break;
        }
    }
    return g;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("NSL_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// NSL_OCT_DENSE=1: OCT through the fused dense build (the A/B baseline of the staged build)
static bool oct_dense_forced() {
    static const bool on = [] {
        const char* e = getenv("NSL_OCT_DENSE");
        return e && e[0] == '1';
    }();
    return on;
}
// The raw grid as a 3-D TMA tensor (x fastest) with a (36, 9, B+1) box; false (-> the cp.async
// staging) when the driver entry point is missing, the base is not 16-B aligned, the x pitch is
// not a multiple of 16 B (n_x % 4 != 0), or the encode fails.  NSL_BUILD_TMA=0 forces cp.async.
static bool encode_raw_map(CUtensorMap& map, const float* raw, int nx, int ny, int nz, int B) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        const char* e = getenv("NSL_BUILD_TMA");
        if (e && e[0] == '0') return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    memset(&map, 0, sizeof map);
    if (!encode || reinterpret_cast<uintptr_t>(raw) % 16 || nx % 4) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    const cuuint64_t strides[2] = {(cuuint64_t)nx * 4, (cuuint64_t)nx * ny * 4};
    const cuuint32_t box[3] = {(cuuint32_t)kStRw, (cuuint32_t)(kStTy + 1), (cuuint32_t)(B + 1)};
    const cuuint32_t es[3] = {1, 1, 1};
    return encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(raw), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool staged_oct_build(int layout, const OccGeom& g) {
    return layout == kOctF32 && (g.shift == 2 || g.shift == 3) && !oct_dense_forced();
}

// Volume build: one fused launch (layout + occupancy rows), then the PDL-launched finalize;
// OCT with 4^3 / 8^3 blocks: occ_reset, the staged occupancy-gated build (PDL), the finalize.
cudaError_t launch_volume_build(const float* raw, const VolDesc& v, void* storage, uint32_t* scratch,
                                unsigned long long* invalid, cudaStream_t s) {
    Raw r{raw, v.nx, v.ny, v.nz};
    if (staged_oct_build(v.layout, v.og)) {
        const int reset_n = v.og.words + v.og.rows;
        occ_reset_kernel<<<(reset_n + 255) / 256 < 1024 ? (reset_n + 255) / 256 : 1024, 256, 0, s>>>(
            v.og, const_cast<uint32_t*>(v.occ), scratch);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        const int tiles_x = (v.nx + 1 + kStTx - 1) / kStTx, tiles_y = (v.ny + 1 + kStTy - 1) / kStTy;
        const int B = 1 << v.og.shift, nlayers = (v.nz + 1 + B - 1) / B, per = 8 / B;   // >= 8 cells of z per CTA
        const dim3 grid((unsigned)(tiles_x * tiles_y), (unsigned)((nlayers + per - 1) / per));
        CUtensorMap map;
        const bool tma = encode_raw_map(map, raw, v.nx, v.ny, v.nz, B);
        float* o = static_cast<float*>(storage);
        uint32_t* mask = const_cast<uint32_t*>(v.occ);
        if (v.og.shift == 2)
            e = tma ? launch_pdl(oct_build_kernel<2, true>, grid, dim3(256), 0, s, map, r, o, v.og, mask, scratch, tiles_x)
                    : launch_pdl(oct_build_kernel<2, false>, grid, dim3(256), 0, s, map, r, o, v.og, mask, scratch, tiles_x);
        else
            e = tma ? launch_pdl(oct_build_kernel<3, true>, grid, dim3(256), 0, s, map, r, o, v.og, mask, scratch, tiles_x)
                    : launch_pdl(oct_build_kernel<3, false>, grid, dim3(256), 0, s, map, r, o, v.og, mask, scratch, tiles_x);
        if (e != cudaSuccess) return e;
        return launch_pdl(occ_finalize_kernel, dim3(1), dim3(kFinThreads), (size_t)v.og.nbz * 16, s, v.og,
                          (const uint32_t*)scratch, const_cast<uint32_t*>(v.occ), const_cast<int32_t*>(v.aabb), invalid);
    }
    const int plane = v.layout == kLinearF32 ? (v.nx + 2) * (v.ny + 2) : (v.nx + 1) * (v.ny + 1);
    const int planes = v.layout == kCornerF16 || v.layout == kOctF32 ? v.nz + 1 : v.nz + 2;
    const bool per_elem = v.layout == kBrickOctF32 || v.layout == kMortonOctF32;   // one thread per element
    const int plane_blocks = per_elem ? (int)((layout_elems(v.layout, v.nx, v.ny, v.nz) + 255) / 256)
                                      : (plane + 255) / 256;
    int kstep = v.layout == kQuadF32  ? (planes + kQuadPlanes - 1) / kQuadPlanes
                : v.layout == kOctF32 ? (planes + kOctRun - 1) / kOctRun
                : per_elem            ? 1
                                      : planes;
    const long max_layout_ctas = 2000000000L - v.og.rows;
    if ((long)plane_blocks * kstep > max_layout_ctas) kstep = (int)(max_layout_ctas / plane_blocks);
    const unsigned grid = (unsigned)(v.og.rows + (long)plane_blocks * kstep);
    const int occ_stride = (int)(grid / (unsigned)v.og.rows);
    const size_t smem = (size_t)v.og.rowwords * 4;
    switch (v.layout) {
        case kLinearF32:
            volume_build_kernel<kLinearF32><<<grid, 256, smem, s>>>(r, storage, v.og, scratch, plane_blocks, kstep,
                                                                          occ_stride);
            break;
        case kQuadF32:
            volume_build_kernel<kQuadF32><<<grid, 256, smem, s>>>(r, storage, v.og, scratch, plane_blocks, kstep,
                                                                          occ_stride);
            break;
        case kCornerF16:
            volume_build_kernel<kCornerF16><<<grid, 256, smem, s>>>(r, storage, v.og, scratch, plane_blocks, kstep,
                                                                          occ_stride);
            break;
        case kOctF32:
            volume_build_kernel<kOctF32><<<grid, 256, smem, s>>>(r, storage, v.og, scratch, plane_blocks, kstep,
                                                                          occ_stride);
            break;
        case kBrickOctF32:
            volume_build_kernel<kBrickOctF32><<<grid, 256, smem, s>>>(r, storage, v.og, scratch, plane_blocks, kstep,
                                                                          occ_stride);
            break;
        case kMortonOctF32:
            volume_build_kernel<kMortonOctF32><<<grid, 256, smem, s>>>(r, storage, v.og, scratch, plane_blocks,
                                                                           kstep, occ_stride);
            break;
        case kTex3dF32:
            volume_build_kernel<kTex3dF32><<<grid, 256, smem, s>>>(
                r, reinterpret_cast<void*>((uintptr_t)v.surf), v.og, scratch, plane_blocks, kstep, occ_stride);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const unsigned fin_ctas = 1u + (unsigned)((v.og.words + kFinThreads / 32 - 1) / (kFinThreads / 32));
    return launch_pdl(occ_finalize_kernel, dim3(fin_ctas), dim3(kFinThreads), (size_t)v.og.nbz * 16, s, v.og, (const uint32_t*)scratch,
                      const_cast<uint32_t*>(v.occ), const_cast<int32_t*>(v.aabb), invalid);
}

}  // namespace nsl
