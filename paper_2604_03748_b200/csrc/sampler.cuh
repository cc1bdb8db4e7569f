// sampler.cuh — device code shared by the march (march.cu) and the six-way bake
// (bake.cu): build-variant switches, the C1 trilinear sampler with the exact
// occupancy skip, the C4 hash, ray/slab helpers and the exact C8 light counts.
// Included inside each translation unit's anonymous namespace usage below.
#pragma once
#include <cuda_fp16.h>

// NSL_CHECK=1 builds a checked library (scripts/gpu_checked.sh): device asserts on every
// volume/mask/lattice index the kernels compute (there is no compute-sanitizer on the pool).
#ifndef NSL_CHECK
#define NSL_CHECK 0
#endif
#if NSL_CHECK
#include <cassert>
#define NSL_ASSERT(c) assert(c)
#else
#define NSL_ASSERT(c) ((void)0)
#endif

#include "nsl_internal.cuh"

namespace nsl {
namespace {

#ifndef NSL_TILEW
#define NSL_TILEW 16     // CTA tile NSL_TILEW x NSL_TILEH pixels, one thread per pixel
#endif
#ifndef NSL_TILEH
#define NSL_TILEH 8      // 16 x 8 -> 128 threads (measured best; 16 x 16 -> 256)
#endif
#ifndef NSL_WARPW
#define NSL_WARPW 8      // warp footprint NSL_WARPW x (32 / NSL_WARPW) pixels (8 x 4 measured best)
#endif
constexpr int kTileW = NSL_TILEW, kTileH = NSL_TILEH, kThreads = NSL_TILEW * NSL_TILEH;
constexpr int kWarpW = NSL_WARPW, kWarpH = 32 / NSL_WARPW, kWarpsX = NSL_TILEW / NSL_WARPW;
static_assert(kThreads % 32 == 0 && NSL_TILEW % NSL_WARPW == 0 && NSL_TILEH % (32 / NSL_WARPW) == 0,
              "CTA tile must be a whole number of warp footprints");
#ifndef NSL_MINB
#define NSL_MINB 5   // min resident CTAs per SM requested from ptxas (register cap = 65536 / (256 * NSL_MINB));
                     // 5 (<= 51 registers, 40 warps/SM) measured fastest on C2 (profiles/r1_sweep.txt)
#endif
#ifndef NSL_VOL_EVF
#define NSL_VOL_EVF 2   // OCT gathers: 2 = L1::no_allocate (the gathers' lines do not displace the mask, frame
                        // constants and spill lines: C2 -1.0 %, C3 -2.1 %, C5 -4.3 % vs evict_first,
                        // profiles/r2_ab17), 1 = L1::evict_first, 0 = plain, 3 = no_allocate + L2::evict_last
                        // (the same as 2, profiles/r2_ab19)
#endif
#ifndef NSL_G3
#define NSL_G3 1    // FAST guide-set (3 lights) launches use the march specialised for it
#endif
#ifndef NSL_L1                  // march specialised for a single light
#define NSL_L1 1
#endif
#ifndef NSL_TV_NL               // the single-light kernel for the TV light model too
#define NSL_TV_NL 1
#endif
#ifndef NSL_TV_G3               // the guide-set kernel for the TV light model
#define NSL_TV_G3 1
#endif
#ifndef NSL_MINB_G3TV
#define NSL_MINB_G3TV 5 // its register cap (48)
#endif
#ifndef NSL_MINB_L1
#define NSL_MINB_L1 6   // its register cap
#endif
#ifndef NSL_MINB_G3
#define NSL_MINB_G3 6   // its register cap (40: 48 warps/SM)
#endif
#ifndef NSL_HZ                  // horizontal guide pair: z plane hoisted out of the light loop
#define NSL_HZ 1
#endif
#ifndef NSL_TILE_RANGE          // FAST/COUNTED ortho: primary steps limited to the tile's occupied-slab range
#define NSL_TILE_RANGE 1
#endif
constexpr int kFast = 0, kDebug = 1, kCounted = 2;

struct Vol {
    const void* __restrict__ data;
    const uint32_t* __restrict__ occ;   // occupancy region (mask | slab boxes), read through the read-only path
    int sy, sz;
    int shift, nbx, nby;
    float sx1, sy1, sz1;          // support upper bounds n+1
    int mask_words;               // NSL_CHECK only: occupancy mask words
};

__device__ __forceinline__ float lerpf(float a, float b, float t) { return __fmaf_rn(t, b - a, a); }

__device__ __forceinline__ bool inside(const Vol& v, float x, float y, float z) {
    return x > 0.0f && x < v.sx1 && y > 0.0f && y < v.sy1 && z > 0.0f && z < v.sz1;
}

// C1 trilinear at an in-support padded-index position (corners always exist
// thanks to the apron).  floor and fraction are exact in fp32.  Samples in an
// empty occupancy block return 0 without touching global memory.
// floor on the FMA pipe: for 0 <= x < 2^22, x + 1.5*2^23 rounded toward -inf is
// exactly floor(x) + 1.5*2^23 (unit spacing there), so the integer sits in the
// low mantissa bits and r - 1.5*2^23 is floor(x) exactly.  No F2I/FRND (the
// quarter-rate XU pipe) per sample.  Positions in support satisfy 0 < x < n+1.
constexpr float kFloorBias = 12582912.0f;   // 1.5 * 2^23, bit pattern 0x4B400000
// C1 trilinear from the gathered corners of element e (cell floors ix, iy, iz) with the exact
// fractions (fx, fy, fz): one load per layout as DESIGN.md §6 describes.
template <int LAYOUT>
__device__ __forceinline__ float gather_interp(const Vol& v, int e, float fx, float fy, float fz) {
    if (LAYOUT == kLinearF32) {
        const float* p = static_cast<const float*>(v.data) + e;
        const float c000 = __ldg(p), c100 = __ldg(p + 1);
        const float c010 = __ldg(p + v.sy), c110 = __ldg(p + v.sy + 1);
        const float c001 = __ldg(p + v.sz), c101 = __ldg(p + v.sz + 1);
        const float c011 = __ldg(p + v.sz + v.sy), c111 = __ldg(p + v.sz + v.sy + 1);
        const float x00 = lerpf(c000, c100, fx), x10 = lerpf(c010, c110, fx);
        const float x01 = lerpf(c001, c101, fx), x11 = lerpf(c011, c111, fx);
        return lerpf(lerpf(x00, x10, fy), lerpf(x01, x11, fy), fz);
    } else if (LAYOUT == kQuadF32) {
        const float4* p = static_cast<const float4*>(v.data) + e;
        const float4 q0 = __ldg(p), q1 = __ldg(p + v.sz);     // (c0, c1 - c0, c2, c3 - c2)
        const float x00 = __fmaf_rn(fx, q0.y, q0.x), x10 = __fmaf_rn(fx, q0.w, q0.z);
        const float x01 = __fmaf_rn(fx, q1.y, q1.x), x11 = __fmaf_rn(fx, q1.w, q1.z);
        return lerpf(lerpf(x00, x10, fy), lerpf(x01, x11, fy), fz);
    } else if (LAYOUT == kOctF32 || LAYOUT == kBrickOctF32 || LAYOUT == kMortonOctF32) {
        // one 256-bit gather: (c000, c100 - c000, c010, c110 - c010 | the same for plane k+1)
        float a0, a1, a2, a3, b0, b1, b2, b3;
#if NSL_VOL_EVF == 3
        asm("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
            : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(b0), "=f"(b1), "=f"(b2), "=f"(b3)
            : "l"(static_cast<const float*>(v.data) + 8 * (size_t)e));
#elif NSL_VOL_EVF == 2
        asm("ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
            : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(b0), "=f"(b1), "=f"(b2), "=f"(b3)
            : "l"(static_cast<const float*>(v.data) + 8 * (size_t)e));
#elif NSL_VOL_EVF
        asm("ld.global.nc.L1::evict_first.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
            : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(b0), "=f"(b1), "=f"(b2), "=f"(b3)
            : "l"(static_cast<const float*>(v.data) + 8 * (size_t)e));
#else
        asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
            : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(b0), "=f"(b1), "=f"(b2), "=f"(b3)
            : "l"(static_cast<const float*>(v.data) + 8 * (size_t)e));
#endif
        const float x00 = __fmaf_rn(fx, a1, a0), x10 = __fmaf_rn(fx, a3, a2);
        const float x01 = __fmaf_rn(fx, b1, b0), x11 = __fmaf_rn(fx, b3, b2);
        return lerpf(lerpf(x00, x10, fy), lerpf(x01, x11, fy), fz);
    } else {
        const uint4 u = __ldg(static_cast<const uint4*>(v.data) + e);
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
        const float2 bb = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
        const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&u.z));
        const float2 d = __half22float2(*reinterpret_cast<const __half2*>(&u.w));
        const float x00 = lerpf(a.x, a.y, fx), x10 = lerpf(bb.x, bb.y, fx);
        const float x01 = lerpf(c.x, c.y, fx), x11 = lerpf(d.x, d.y, fx);
        return lerpf(lerpf(x00, x10, fy), lerpf(x01, x11, fy), fz);
    }
}

// Element index of cell (ix, iy, iz) for the element-addressed layouts (z part zpart, zlow
// precomputed by zplane for horizontal lines; TEX3D has no element index).
__device__ __forceinline__ int spread3(int a) {   // bits b2 b1 b0 -> b2 0 0 b1 0 0 b0
    return (a & 1) | ((a & 2) << 2) | ((a & 4) << 4);
}
template <int LAYOUT>
__device__ __forceinline__ int elem_index(const Vol& v, int ix, int iy, int zpart, int zlow) {
    if (LAYOUT == kBrickOctF32) return ((zpart + (iy >> 2) * v.sy + (ix >> 2)) << 6) | zlow | ((iy & 3) << 2) | (ix & 3);
    if (LAYOUT == kMortonOctF32) return ((zpart + (iy >> 3) * v.sy + (ix >> 3)) << 9) | zlow | (spread3(iy & 7) << 1) |
                                        spread3(ix & 7);
    return ix + iy * v.sy + zpart;
}
template <int LAYOUT>
__device__ __forceinline__ int zpart_of(const Vol& v, int iz) {
    return LAYOUT == kBrickOctF32 ? (iz >> 2) * v.sz : LAYOUT == kMortonOctF32 ? (iz >> 3) * v.sz : iz * v.sz;
}
template <int LAYOUT>
__device__ __forceinline__ int zlow_of(int iz) {
    return LAYOUT == kBrickOctF32 ? (iz & 3) << 4 : LAYOUT == kMortonOctF32 ? spread3(iz & 7) << 2 : 0;
}

// TEX3D: the QUAD float4 of cells (ix, iy, iz) and (ix, iy, iz + 1) by two point-sampled fetches
// (texel t covers [t, t + 1): the coordinate floor + 0.5 selects it exactly), then QUAD's lerps.
__device__ __forceinline__ float gather_tex3d(const Vol& v, float flx, float fly, float flz, float fx, float fy,
                                              float fz) {
    const cudaTextureObject_t t = (cudaTextureObject_t) reinterpret_cast<uintptr_t>(v.data);
    const float cx = __fadd_rn(flx, 0.5f), cy = __fadd_rn(fly, 0.5f), cz = __fadd_rn(flz, 0.5f);
    const float4 q0 = tex3D<float4>(t, cx, cy, cz), q1 = tex3D<float4>(t, cx, cy, __fadd_rn(cz, 1.0f));
    const float x00 = __fmaf_rn(fx, q0.y, q0.x), x10 = __fmaf_rn(fx, q0.w, q0.z);
    const float x01 = __fmaf_rn(fx, q1.y, q1.x), x11 = __fmaf_rn(fx, q1.w, q1.z);
    return lerpf(lerpf(x00, x10, fy), lerpf(x01, x11, fy), fz);
}

template <int LAYOUT, bool COUNT>
__device__ __forceinline__ float sample(const Vol& v, float x, float y, float z, uint32_t& gathers) {
    // cell floors (shared with the gather below), block = cell >> shift
    const float rx = __fadd_rd(x, kFloorBias), ry = __fadd_rd(y, kFloorBias), rz = __fadd_rd(z, kFloorBias);
    const int ix = __float_as_int(rx) - 0x4B400000, iy = __float_as_int(ry) - 0x4B400000,
              iz = __float_as_int(rz) - 0x4B400000;
    const int b = ((iz >> v.shift) * v.nby + (iy >> v.shift)) * v.nbx + (ix >> v.shift);
    NSL_ASSERT(ix >= 0 && iy >= 0 && iz >= 0 && (float)ix < v.sx1 && (float)iy < v.sy1 && (float)iz < v.sz1);
    NSL_ASSERT(b >= 0 && (b >> 5) < v.mask_words);
    const uint32_t word = __ldg(v.occ + (b >> 5));
    if (!((word >> (b & 31)) & 1u)) return 0.0f;
    if (COUNT) ++gathers;
    const float flx = __fsub_rn(rx, kFloorBias), fly = __fsub_rn(ry, kFloorBias), flz = __fsub_rn(rz, kFloorBias);
    const float fx = __fsub_rn(x, flx), fy = __fsub_rn(y, fly), fz = __fsub_rn(z, flz);
    if constexpr (LAYOUT == kTex3dF32) return gather_tex3d(v, flx, fly, flz, fx, fy, fz);
    else return gather_interp<LAYOUT>(v, elem_index<LAYOUT>(v, ix, iy, zpart_of<LAYOUT>(v, iz), zlow_of<LAYOUT>(iz)),
                                      fx, fy, fz);
}

// A horizontal light line (L_z == 0 bit-exactly: every Y_j keeps U_z, since fma(s, 0, u_z) ==
// u_z) shares one z cell, fraction and block row: computed once per occupied primary sample
// instead of per light sample.  sample_hz(v, zp, x, y) == sample(v, x, y, z) bit for bit.
struct ZPlane {
    int zb;      // (iz >> shift) * nby: the block row base
    int ze;      // the z part of the element index (zpart_of)
    int zl;      // the z bits inside a brick / tile (zlow_of)
    float flz, fz;
};
template <int LAYOUT>
__device__ __forceinline__ ZPlane zplane(const Vol& v, float z) {
    const float rz = __fadd_rd(z, kFloorBias);
    const int iz = __float_as_int(rz) - 0x4B400000;
    ZPlane p;
    p.zb = (iz >> v.shift) * v.nby;
    p.ze = zpart_of<LAYOUT>(v, iz);
    p.zl = zlow_of<LAYOUT>(iz);
    p.flz = __fsub_rn(rz, kFloorBias);
    p.fz = __fsub_rn(z, p.flz);
    return p;
}
template <int LAYOUT, bool COUNT>
__device__ __forceinline__ float sample_hz(const Vol& v, const ZPlane& zp, float x, float y, uint32_t& gathers) {
    const float rx = __fadd_rd(x, kFloorBias), ry = __fadd_rd(y, kFloorBias);
    const int ix = __float_as_int(rx) - 0x4B400000, iy = __float_as_int(ry) - 0x4B400000;
    const int b = (zp.zb + (iy >> v.shift)) * v.nbx + (ix >> v.shift);
    NSL_ASSERT(ix >= 0 && iy >= 0 && (float)ix < v.sx1 && (float)iy < v.sy1);
    NSL_ASSERT(b >= 0 && (b >> 5) < v.mask_words);
    const uint32_t word = __ldg(v.occ + (b >> 5));
    if (!((word >> (b & 31)) & 1u)) return 0.0f;
    if (COUNT) ++gathers;
    const float flx = __fsub_rn(rx, kFloorBias), fly = __fsub_rn(ry, kFloorBias);
    const float fx = __fsub_rn(x, flx), fy = __fsub_rn(y, fly);
    if constexpr (LAYOUT == kTex3dF32) return gather_tex3d(v, flx, fly, zp.flz, fx, fy, zp.fz);
    else return gather_interp<LAYOUT>(v, elem_index<LAYOUT>(v, ix, iy, zp.ze, zp.zl), fx, fy, zp.fz);
}

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

// C4: hash chain keyed by (seed, frame, pixel)
__device__ __forceinline__ uint32_t jitter_hash(uint32_t seed_lo, uint32_t seed_hi, uint32_t frame, uint32_t pixel) {
    uint32_t h = fmix32(seed_lo ^ 0x9E3779B9u);
    h = fmix32(h ^ seed_hi);
    h = fmix32(h ^ frame);
    return fmix32(h ^ pixel);
}
__device__ __forceinline__ float jitter_delta(uint32_t h32, float h) {
    const float u = __fmul_rn(__uint2float_rn(h32 >> 8), 5.9604644775390625e-08f);  // exact: 24-bit int * 2^-24
    return __fmul_rn(u, h);
}

struct Ray {
    float ox, oy, oz, dx, dy, dz, delta, h;
    __device__ __forceinline__ void at(int n, float& t, float& x, float& y, float& z) const {
        atf((float)n, t, x, y, z);
    }
    __device__ __forceinline__ void atf(float nf, float& t, float& x, float& y, float& z) const {
        t = __fmaf_rn(nf, h, delta);
        x = __fmaf_rn(t, dx, ox);
        y = __fmaf_rn(t, dy, oy);
        z = __fmaf_rn(t, dz, oz);
    }
    __device__ __forceinline__ bool in(const Vol& v, int n) const {
        float t, x, y, z;
        at(n, t, x, y, z);
        return inside(v, x, y, z);
    }
};

// inv: 1/d (per-frame constant for orthographic cameras, computed per ray otherwise)
__device__ __forceinline__ void slab(float o, float d, float inv, float s, float eps, float& t0, float& t1,
                                     bool& miss) {
    if (d != 0.0f) {
        float ta = (-eps - o) * inv, tb = (s + eps - o) * inv;
        if (ta > tb) {
            const float tt = ta;
            ta = tb;
            tb = tt;
        }
        t0 = fmaxf(t0, ta);
        t1 = fminf(t1, tb);
    } else if (!(o > -eps && o < s + eps)) {
        miss = true;
    }
}

// C5: exact first/last in-support step in [1, Ncap] (0,-1 if none).  A float
// slab test on the box expanded by 1e-3 index units brackets the range to
// within one step; exact per-sample tests then shrink it (the in-support set
// is contiguous because every coordinate is monotone in n).
__device__ __forceinline__ void clip_ray(const Ray& r, const Vol& v, const float inv[3], float inv_h, int Ncap,
                                         int& n0, int& n1) {
    n0 = 0;
    n1 = -1;
    const float eps = 1e-3f;
    float t0 = -3.0e38f, t1 = 3.0e38f;
    bool miss = false;
    slab(r.ox, r.dx, inv[0], v.sx1, eps, t0, t1, miss);
    slab(r.oy, r.dy, inv[1], v.sy1, eps, t0, t1, miss);
    slab(r.oz, r.dz, inv[2], v.sz1, eps, t0, t1, miss);
    if (miss || !(t0 <= t1)) return;
    float a = floorf((t0 - r.delta) * inv_h) - 1.0f, b = ceilf((t1 - r.delta) * inv_h) + 1.0f;
    a = fmaxf(a, 1.0f);
    b = fminf(b, (float)Ncap);
    if (!(a <= b)) return;
    int na = (int)a, nb = (int)b;
    while (na <= nb && !r.in(v, na)) ++na;
    while (nb >= na && !r.in(v, nb)) --nb;
    if (na > nb) return;
    n0 = na;
    n1 = nb;
}

// C8: M = number of leading in-support light samples Y_j = fma(j*h_l, L, U).
// lim/ilh: per-frame exit plane and 1/(L*h_l) per axis (FrameParams) -> estimate, then exact fix-up.
__device__ __forceinline__ int light_count(const Vol& v, float ux, float uy, float uz, float lx, float ly, float lz,
                                           float hl, const float lim[3], const float ilh[3]) {
    const float m = fminf(fminf((lim[0] - ux) * ilh[0], (lim[1] - uy) * ilh[1]), (lim[2] - uz) * ilh[2]);
    const float mf = fminf(fmaxf(floorf(m), 0.0f), 16777216.0f);
    int M = (int)mf;
    auto in_j = [&](int j) {
        const float s = __fmul_rn((float)j, hl);
        return inside(v, __fmaf_rn(s, lx, ux), __fmaf_rn(s, ly, uy), __fmaf_rn(s, lz, uz));
    };
    while (M > 0 && !in_j(M)) --M;
    while (in_j(M + 1)) ++M;
    return M;
}

// sum of rho over j = 1..M along the light (all in support); two independent
// accumulators give the scheduler two gathers in flight per thread.
template <int LAYOUT, bool COUNT>
__device__ __forceinline__ float light_sum(const Vol& v, float ux, float uy, float uz, float lx, float ly, float lz,
                                           float hl, int M, uint32_t& gathers) {
    float acc0 = 0.0f, acc1 = 0.0f;
    int j = 1;
    float jf = 1.0f;   // exact float copy of j (j < 2^24): no I2F in the loop
    for (; j + 1 <= M; j += 2, jf += 2.0f) {
        const float s0 = __fmul_rn(jf, hl), s1 = __fmul_rn(jf + 1.0f, hl);
        acc0 += sample<LAYOUT, COUNT>(v, __fmaf_rn(s0, lx, ux), __fmaf_rn(s0, ly, uy), __fmaf_rn(s0, lz, uz), gathers);
        acc1 += sample<LAYOUT, COUNT>(v, __fmaf_rn(s1, lx, ux), __fmaf_rn(s1, ly, uy), __fmaf_rn(s1, lz, uz), gathers);
    }
    if (j <= M) {
        const float s0 = __fmul_rn(jf, hl);
        acc0 += sample<LAYOUT, COUNT>(v, __fmaf_rn(s0, lx, ux), __fmaf_rn(s0, ly, uy), __fmaf_rn(s0, lz, uz), gathers);
    }
    return acc0 + acc1;
}

// The guide set's top and bottom lights are exact opposites (L_g,2 = -L_g,1 bit
// for bit): both marches walk the same line through U in opposite directions.
// One loop serves both: s_j is shared and fma(-s, L, U) == fma(s, -L, U) exactly,
// so the positions are the canonical ones of C8 for each light.
template <int LAYOUT, bool COUNT>
__device__ __forceinline__ void light_sum_pair(const Vol& v, float ux, float uy, float uz, float lx, float ly,
                                               float lz, float hl, int Ma, int Mb, float& sa, float& sb,
                                               uint32_t& gathers) {
    float a = 0.0f, b = 0.0f;
    const int M = max(Ma, Mb);
    float jf = 1.0f;
    for (int j = 1; j <= M; ++j, jf += 1.0f) {
        const float s = __fmul_rn(jf, hl);
        if (j <= Ma) a += sample<LAYOUT, COUNT>(v, __fmaf_rn(s, lx, ux), __fmaf_rn(s, ly, uy), __fmaf_rn(s, lz, uz), gathers);
        if (j <= Mb)
            b += sample<LAYOUT, COUNT>(v, __fmaf_rn(-s, lx, ux), __fmaf_rn(-s, ly, uy), __fmaf_rn(-s, lz, uz), gathers);
    }
    sa = a;
    sb = b;
}

// light_sum_pair for a horizontal pair (both lights' L_z == 0 bit-exactly): the same samples
// through sample_hz, the z plane of U computed once.
#ifndef NSL_ZPIN
#define NSL_ZPIN 1
#endif
template <int LAYOUT, bool COUNT>
__device__ __forceinline__ void light_sum_pair_hz(const Vol& v, float ux, float uy, float uz, float lx, float ly,
                                                  float hl, int Ma, int Mb, float& sa, float& sb, uint32_t& gathers) {
#if NSL_ZPIN
    // opaque copies: ptxas must keep the plane in registers instead of recomputing it per sample
    ZPlane zp = zplane<LAYOUT>(v, uz);
    asm volatile("" : "+r"(zp.zb), "+r"(zp.ze), "+f"(zp.fz));
#else
    const ZPlane zp = zplane<LAYOUT>(v, uz);
#endif
    float a = 0.0f, b = 0.0f;
    const int M = max(Ma, Mb);
    float jf = 1.0f;
    for (int j = 1; j <= M; ++j, jf += 1.0f) {
        const float s = __fmul_rn(jf, hl);
        if (j <= Ma) a += sample_hz<LAYOUT, COUNT>(v, zp, __fmaf_rn(s, lx, ux), __fmaf_rn(s, ly, uy), gathers);
        if (j <= Mb) b += sample_hz<LAYOUT, COUNT>(v, zp, __fmaf_rn(-s, lx, ux), __fmaf_rn(-s, ly, uy), gathers);
    }
    sa = a;
    sb = b;
}

// Fast-path bound on the light samples that can be nonzero: the estimate of the
// region count plus one (>= the exact count of in-region samples), then shrunk with exact prescribed-op tests until the last sample is in
// support (so every index is valid).  Every in-support sample inside the
// occupied box is covered, hence the sum equals the canonical one (C8).
// The region (occupied box or slab box) lies inside the support on every axis and the
// estimate (plane - u) * ilh is monotone in the plane, so the region's estimate is never
// above the support's: it alone bounds the count.
__device__ __forceinline__ int light_bound(const Vol& v, float ux, float uy, float uz, float lx, float ly, float lz,
                                           float hl, const float ilh[3], const float alim[3]) {
    const float mb = fminf(fminf((alim[0] - ux) * ilh[0], (alim[1] - uy) * ilh[1]), (alim[2] - uz) * ilh[2]);
    float m = floorf(mb) + 1.0f;
    m = fminf(fmaxf(m, 0.0f), 16777216.0f);
    while (m > 0.0f) {
        const float s = __fmul_rn(m, hl);
        if (inside(v, __fmaf_rn(s, lx, ux), __fmaf_rn(s, ly, uy), __fmaf_rn(s, lz, uz))) break;
        m -= 1.0f;
    }
    return (int)m;
}

// Conservative count of leading light samples inside the occupied box (one
// extra for rounding): samples beyond it are exactly 0 and need not be taken.
__device__ __forceinline__ int box_count(float ux, float uy, float uz, const float alim[3], const float ilh[3]) {
    const float m = fminf(fminf((alim[0] - ux) * ilh[0], (alim[1] - uy) * ilh[1]), (alim[2] - uz) * ilh[2]);
    return (int)fminf(fmaxf(floorf(m), -1.0f), 16777215.0f) + 1;
}

// Exit planes of the region that can hold nonzero samples of light l's march from
// height uz: for a horizontal light (L_z == 0 exactly, so every Y_j,z == uz and the
// march stays in the z block-slab of uz) the slab's 2-D box of non-empty blocks;
// otherwise the occupied 3-D box.  Either way samples beyond it are exactly 0.
__device__ __forceinline__ void march_region(const FrameParams& sp, const Vol& v, int l, float uz, float out[3]) {
    if ((sp.lz0 >> l) & 1) {
        const int iz = __float_as_int(__fadd_rd(uz, kFloorBias)) - 0x4B400000;
        const int bz = iz >> v.shift;
        const int* slab = reinterpret_cast<const int*>(v.occ) + sp.slab_off;
        const int2 mn = __ldg(reinterpret_cast<const int2*>(slab + 2 * bz));
        const int2 mx = __ldg(reinterpret_cast<const int2*>(slab + 2 * sp.occ_nbz + 2 * bz));
        const float B = (float)(1 << v.shift);
        const float lox = (float)mn.x * B, hix = fminf((float)(mx.x + 1) * B, v.sx1);
        const float loy = (float)mn.y * B, hiy = fminf((float)(mx.y + 1) * B, v.sy1);
        const float Lx = sp.Lg[l][0], Ly = sp.Lg[l][1];
        out[0] = Lx > 0.0f ? hix : (Lx < 0.0f ? lox : 3.0e38f);
        out[1] = Ly > 0.0f ? hiy : (Ly < 0.0f ? loy : 3.0e38f);
        out[2] = 3.0e38f;
    } else {
        out[0] = sp.alim[l][0];
        out[1] = sp.alim[l][1];
        out[2] = sp.alim[l][2];
    }
}

// The guide pair's two regions (L_g,2 = -L_g,1 bit-exactly, so light 2's exit plane on each
// axis is light 1's other one): for horizontal lights one slab-box load serves both; otherwise
// the occupied box.  Equal to march_region(sp, v, 1, uz) and march_region(sp, v, 2, uz).
__device__ __forceinline__ void pair_regions(const FrameParams& sp, const Vol& v, float uz, float ra[3],
                                             float rb[3]) {
    const float Lx = sp.Lg[1][0], Ly = sp.Lg[1][1];
    if ((sp.lz0 >> 1) & 1) {
        const int iz = __float_as_int(__fadd_rd(uz, kFloorBias)) - 0x4B400000;
        const int bz = iz >> v.shift;
        const int* slab = reinterpret_cast<const int*>(v.occ) + sp.slab_off;
        const int2 mn = __ldg(reinterpret_cast<const int2*>(slab + 2 * bz));
        const int2 mx = __ldg(reinterpret_cast<const int2*>(slab + 2 * sp.occ_nbz + 2 * bz));
        const float B = (float)(1 << v.shift);
        const float lox = (float)mn.x * B, hix = fminf((float)(mx.x + 1) * B, v.sx1);
        const float loy = (float)mn.y * B, hiy = fminf((float)(mx.y + 1) * B, v.sy1);
        ra[0] = Lx > 0.0f ? hix : (Lx < 0.0f ? lox : 3.0e38f);
        rb[0] = Lx > 0.0f ? lox : (Lx < 0.0f ? hix : 3.0e38f);
        ra[1] = Ly > 0.0f ? hiy : (Ly < 0.0f ? loy : 3.0e38f);
        rb[1] = Ly > 0.0f ? loy : (Ly < 0.0f ? hiy : 3.0e38f);
        ra[2] = rb[2] = 3.0e38f;
    } else {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            ra[q] = sp.alim[1][q];
            rb[q] = sp.alim[2][q];
        }
    }
}

// pair_regions from the packed per-frame constants (FrameParams.pk_geo = (slab_off, occ_nbz, lz0,
// pair12) and light 1's (Lx, Ly)): the same values, fewer loads.
__device__ __forceinline__ void pair_regions_pk(const FrameParams& sp, const Vol& v, float uz, int4 geo, float Lx,
                                                float Ly, float ra[3], float rb[3]) {
    if ((geo.z >> 1) & 1) {
        const int iz = __float_as_int(__fadd_rd(uz, kFloorBias)) - 0x4B400000;
        const int bz = iz >> v.shift;
        const int* slab = reinterpret_cast<const int*>(v.occ) + geo.x;
        const int2 mn = __ldg(reinterpret_cast<const int2*>(slab + 2 * bz));
        const int2 mx = __ldg(reinterpret_cast<const int2*>(slab + 2 * geo.y + 2 * bz));
        const float B = (float)(1 << v.shift);
        const float lox = (float)mn.x * B, hix = fminf((float)(mx.x + 1) * B, v.sx1);
        const float loy = (float)mn.y * B, hiy = fminf((float)(mx.y + 1) * B, v.sy1);
        ra[0] = Lx > 0.0f ? hix : (Lx < 0.0f ? lox : 3.0e38f);
        rb[0] = Lx > 0.0f ? lox : (Lx < 0.0f ? hix : 3.0e38f);
        ra[1] = Ly > 0.0f ? hiy : (Ly < 0.0f ? loy : 3.0e38f);
        rb[1] = Ly > 0.0f ? loy : (Ly < 0.0f ? hiy : 3.0e38f);
        ra[2] = rb[2] = 3.0e38f;
    } else {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            ra[q] = sp.alim[1][q];
            rb[q] = sp.alim[2][q];
        }
    }
}

__device__ __forceinline__ float hg32(float g, float c) {
    const float d = (1.0f + g * g) - 2.0f * g * c;
    return (1.0f - g * g) / (12.566370614359172f * d * sqrtf(d));
}


}  // namespace
}  // namespace nsl
