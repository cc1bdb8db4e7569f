// march.cu — rows a2, a4-a8: the guiding-map ray march (Algorithm 1,
// L394-407; C3-C12) for sm_100a.
//
// One thread per pixel; a warp marches a coherent 8x4 pixel tile, a CTA a
// 16x16 tile (8 warps); blockIdx.z is the frame of the batch (row a9).
// Sample positions use only explicitly rounded fp32 operations (__fmaf_rn,
// __fmul_rn) so that every index decision is bit-identical to the oracle
// (C14); values are fp32 with FMA lerps.  The step range is
// clipped exactly (C5) and each light march's length is computed exactly
// (C8) so the inner loops carry no bounds tests.
//
// The path is bound by L1 data-pipe wavefronts of the trilinear gathers
// (profiles/).  Before gathering, every sample tests the
// volume's occupancy bitmask, staged per CTA in shared memory: a sample
// whose cell lies in an all-zero block is exactly 0 (C1), so skipping its
// loads changes no bit of the result while removing most of the wavefronts
// (empty space outside the smoke).
#include <cuda_fp16.h>

#include "nsl_internal.cuh"

namespace nsl {
namespace {

#ifndef NSL_TILEH
#define NSL_TILEH 8      // CTA tile 16 x NSL_TILEH pixels (warps of 8x4): 8 -> 128 threads (measured best), 16 -> 256
#endif
constexpr int kTileW = 16, kTileH = NSL_TILEH, kThreads = 2 * NSL_TILEH * 8;
#ifndef NSL_BLOCKIDX
#define NSL_BLOCKIDX 0   // occupancy block index: 1 exact fp32 FMAs, 0 integer shifts of the cell floor (measured equal, profiles/r1_sweep.txt)
#endif
#ifndef NSL_MASKREAD
#define NSL_MASKREAD 0   // mask word read: 1 ld.shared via a 32-bit address, 0 extern shared array
#endif
#ifndef NSL_PAIRWALK
#define NSL_PAIRWALK 1   // paired top/bottom march: 1 combined chord walk, 0 lock-step both sides
#endif
#ifndef NSL_STAGE
#define NSL_STAGE 0      // 1: stage FrameParams + occupancy region in shared memory per CTA; 0: read them
                         //    through the read-only path from global memory (L1-resident; measured equal or
                         //    better, no __syncthreads, all of L1 for the volume)
#endif
#ifndef NSL_MINB
#define NSL_MINB 5   // min resident CTAs per SM requested from ptxas (register cap = 65536 / (256 * NSL_MINB));
                     // 5 (<= 51 registers, 40 warps/SM) measured fastest on C2 (profiles/r1_sweep.txt)
#endif
constexpr int kFast = 0, kDebug = 1, kCounted = 2;

struct Vol {
    const void* __restrict__ data;
    const uint32_t* __restrict__ occ;   // occupancy region in global memory (NSL_STAGE == 0)
    uint32_t mask_sa;             // shared-space byte address of the occupancy mask
    int sy, sz;
    float inv_b, nbx_f, nbxy_f;   // 2^-shift, blocks per x row, blocks per z slab (exact in fp32)
    int shift, nbx, nby;
    float sx1, sy1, sz1;          // support upper bounds n+1
};

// Dynamic shared memory of march_kernel: [FrameParams | occupancy mask words].
// Indexed through this file-scope array so the mask test is one LDS with an
// immediate offset (no generic->shared address conversion in the loops).
extern __shared__ __align__(16) uint32_t nsl_smem[];
#if NSL_STAGE
constexpr int kMaskWord0 = (int)(sizeof(FrameParams) / 4);
#endif

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
#if NSL_BLOCKIDX == 1
__device__ __forceinline__ void cellof(float x, int& i, float& frac) {
    const float r = __fadd_rd(x, kFloorBias);
    i = __float_as_int(r) - 0x4B400000;
    frac = __fsub_rn(x, __fsub_rn(r, kFloorBias));
}
#endif

template <int LAYOUT, bool COUNT>
__device__ __forceinline__ float sample(const Vol& v, float x, float y, float z, uint32_t& gathers) {
#if NSL_BLOCKIDX == 1
    // occupancy block index in exact fp32: floor(x / B) via fma rounded toward -inf
    // onto the 1.5*2^23 grid (x * 2^-s is exact), then the linear index with two
    // exact FMAs (every term is an integer < 2^24); the bias stays in the x term.
    const float bx = __fmaf_rd(x, v.inv_b, kFloorBias);
    const float by = __fsub_rn(__fmaf_rd(y, v.inv_b, kFloorBias), kFloorBias);
    const float bz = __fsub_rn(__fmaf_rd(z, v.inv_b, kFloorBias), kFloorBias);
    const int b = __float_as_int(__fmaf_rn(bz, v.nbxy_f, __fmaf_rn(by, v.nbx_f, bx))) - 0x4B400000;
#else
    // cell floors (shared with the gather below), block = cell >> shift
    const float rx = __fadd_rd(x, kFloorBias), ry = __fadd_rd(y, kFloorBias), rz = __fadd_rd(z, kFloorBias);
    const int ix = __float_as_int(rx) - 0x4B400000, iy = __float_as_int(ry) - 0x4B400000,
              iz = __float_as_int(rz) - 0x4B400000;
    const int b = ((iz >> v.shift) * v.nby + (iy >> v.shift)) * v.nbx + (ix >> v.shift);
#endif
#if NSL_MASKREAD == 1
    uint32_t word;
    asm("ld.shared.u32 %0, [%1];" : "=r"(word) : "r"(v.mask_sa + ((uint32_t)b >> 5) * 4u));
#else
#if NSL_STAGE
    const uint32_t word = nsl_smem[kMaskWord0 + (b >> 5)];
#else
    const uint32_t word = __ldg(v.occ + (b >> 5));
#endif
#endif
    if (!((word >> (b & 31)) & 1u)) return 0.0f;
    if (COUNT) ++gathers;
#if NSL_BLOCKIDX == 1
    int ix, iy, iz;
    float fx, fy, fz;
    cellof(x, ix, fx);
    cellof(y, iy, fy);
    cellof(z, iz, fz);
#else
    const float fx = __fsub_rn(x, __fsub_rn(rx, kFloorBias)), fy = __fsub_rn(y, __fsub_rn(ry, kFloorBias)),
                fz = __fsub_rn(z, __fsub_rn(rz, kFloorBias));
#endif
    const int e = ix + iy * v.sy + iz * v.sz;
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
#if NSL_PAIRWALK == 1
    // Walk the combined chord k = 0 .. Ma+Mb-1 (j = k+1 on the +L side, then j = k-Ma+1
    // on the -L side) two samples per iteration: no lane idles on the shorter side.
    // jf carries the sign of the side, so s = jf*h_l = +-fl(j*h_l) exactly.
    float a = 0.0f, b = 0.0f;
    const int K = Ma + Mb;
    const float maf = (float)Ma;
    float kf = 0.0f;
    int k = 0;
    for (; k + 1 < K; k += 2, kf += 2.0f) {
        const float j0 = kf < maf ? kf + 1.0f : maf - kf - 1.0f;
        const float j1 = kf + 1.0f < maf ? kf + 2.0f : maf - kf - 2.0f;
        const float s0 = __fmul_rn(j0, hl), s1 = __fmul_rn(j1, hl);
        const float r0 = sample<LAYOUT, COUNT>(v, __fmaf_rn(s0, lx, ux), __fmaf_rn(s0, ly, uy), __fmaf_rn(s0, lz, uz), gathers);
        const float r1 = sample<LAYOUT, COUNT>(v, __fmaf_rn(s1, lx, ux), __fmaf_rn(s1, ly, uy), __fmaf_rn(s1, lz, uz), gathers);
        if (j0 > 0.0f) a += r0; else b += r0;
        if (j1 > 0.0f) a += r1; else b += r1;
    }
    if (k < K) {
        const float j0 = kf < maf ? kf + 1.0f : maf - kf - 1.0f;
        const float s0 = __fmul_rn(j0, hl);
        const float r0 = sample<LAYOUT, COUNT>(v, __fmaf_rn(s0, lx, ux), __fmaf_rn(s0, ly, uy), __fmaf_rn(s0, lz, uz), gathers);
        if (j0 > 0.0f) a += r0; else b += r0;
    }
#else
    float a = 0.0f, b = 0.0f;
    const int M = max(Ma, Mb);
    float jf = 1.0f;
    for (int j = 1; j <= M; ++j, jf += 1.0f) {
        const float s = __fmul_rn(jf, hl);
        if (j <= Ma) a += sample<LAYOUT, COUNT>(v, __fmaf_rn(s, lx, ux), __fmaf_rn(s, ly, uy), __fmaf_rn(s, lz, uz), gathers);
        if (j <= Mb)
            b += sample<LAYOUT, COUNT>(v, __fmaf_rn(-s, lx, ux), __fmaf_rn(-s, ly, uy), __fmaf_rn(-s, lz, uz), gathers);
    }
#endif
    sa = a;
    sb = b;
}

// Fast-path bound on the light samples that can be nonzero: the estimate of the
// support count plus one (>= the exact count), capped by the occupied-box
// count, then shrunk with exact prescribed-op tests until the last sample is in
// support (so every index is valid).  Every in-support sample inside the
// occupied box is covered, hence the sum equals the canonical one (C8).
__device__ __forceinline__ int light_bound(const Vol& v, float ux, float uy, float uz, float lx, float ly, float lz,
                                           float hl, const float lim[3], const float ilh[3], const float alim[3]) {
    const float ms = fminf(fminf((lim[0] - ux) * ilh[0], (lim[1] - uy) * ilh[1]), (lim[2] - uz) * ilh[2]);
    const float mb = fminf(fminf((alim[0] - ux) * ilh[0], (alim[1] - uy) * ilh[1]), (alim[2] - uz) * ilh[2]);
    float m = fminf(floorf(ms), floorf(mb)) + 1.0f;
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
#if NSL_STAGE
        const int* slab = reinterpret_cast<const int*>(nsl_smem) + kMaskWord0 + sp.slab_off;
        const int2 mn = *reinterpret_cast<const int2*>(slab + 2 * bz);
        const int2 mx = *reinterpret_cast<const int2*>(slab + 2 * sp.occ_nbz + 2 * bz);
#else
        const int* slab = reinterpret_cast<const int*>(v.occ) + sp.slab_off;
        const int2 mn = __ldg(reinterpret_cast<const int2*>(slab + 2 * bz));
        const int2 mx = __ldg(reinterpret_cast<const int2*>(slab + 2 * sp.occ_nbz + 2 * bz));
#endif
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

__device__ __forceinline__ float hg32(float g, float c) {
    const float d = (1.0f + g * g) - 2.0f * g * c;
    return (1.0f - g * g) / (12.566370614359172f * d * sqrtf(d));
}

template <int LAYOUT, int PROJ, int MODE>
__global__ void __launch_bounds__(kThreads, NSL_MINB * 256 / kThreads) march_kernel(const FrameParams* __restrict__ fps, const MarchConst mc,
                                                         float4* __restrict__ out_rgbt, float* __restrict__ out_depth,
                                                         uint32_t* __restrict__ out_debug,
                                                         unsigned long long* __restrict__ counters, int W, int H,
                                                         const uint32_t* __restrict__ tile_order, int F) {
    constexpr bool DEBUG = MODE == kDebug, COUNT = MODE == kCounted;
#if NSL_STAGE
    uint4* smem = reinterpret_cast<uint4*>(nsl_smem);
    FrameParams& sp = *reinterpret_cast<FrameParams*>(smem);
    uint4* smask4 = smem + sizeof(FrameParams) / 16;
#endif
    // 1-D grid over (tile rank, frame), frame fastest; tiles in centre-out order
    // (tile_order) so the heavy tiles of every frame start first and the tail of
    // the launch is made of cheap border tiles.
    const int f = (int)(blockIdx.x % (unsigned)F);
    const uint32_t tile = __ldg(tile_order + blockIdx.x / (unsigned)F);
    const int tx = (int)(tile & 0xffffu), ty = (int)(tile >> 16);
#if NSL_STAGE
    {
        const uint4* src = reinterpret_cast<const uint4*>(fps + f);
        for (int i = threadIdx.x; i < (int)(sizeof(FrameParams) / 16); i += blockDim.x) smem[i] = src[i];
    }
    __syncthreads();
#else
    const FrameParams& sp = fps[f];
#endif
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * kTileW + (warp & 1) * 8 + (lane & 7);
    const int py = ty * kTileH + (warp >> 1) * 4 + (lane >> 3);
    const bool valid = px < W && py < H;
    const size_t o = (size_t)f * (size_t)W * (size_t)H + (size_t)py * W + px;

    Vol v;
    v.data = sp.data;
    v.sy = sp.sy;
    v.sz = sp.sz;
#if NSL_STAGE
    v.mask_sa = (uint32_t)__cvta_generic_to_shared(smask4);
#else
    v.mask_sa = 0;
#endif
    v.occ = sp.occ;
    v.inv_b = __int_as_float((127 - sp.occ_shift) << 23);   // 2^-shift exactly
    v.nbx_f = (float)sp.occ_nbx;
    v.nbxy_f = (float)(sp.occ_nbx * sp.occ_nby);
    v.shift = sp.occ_shift;
    v.nbx = sp.occ_nbx;
    v.nby = sp.occ_nby;
    v.sx1 = sp.supp[0];
    v.sy1 = sp.supp[1];
    v.sz1 = sp.supp[2];

    if (PROJ == 0) {
        // Tile culling (exact): every ray of the tile is parallel to D_g with its origin
        // within tile_r of the centre ray; if the centre ray misses the support box
        // expanded by tile_r, no sample of the tile is in support (C5) and the
        // output is the empty map (L = 0, T = 1, D = 0, counters 0).
        const float cx = (float)(tx * kTileW) + 0.5f * (kTileW - 1), cy = (float)(ty * kTileH) + 0.5f * (kTileH - 1);
        Ray c;
        c.ox = fmaf(cy, sp.Ey[0], fmaf(cx, sp.Ex[0], sp.B[0]));
        c.oy = fmaf(cy, sp.Ey[1], fmaf(cx, sp.Ex[1], sp.B[1]));
        c.oz = fmaf(cy, sp.Ey[2], fmaf(cx, sp.Ex[2], sp.B[2]));
        // FAST mode culls against the occupied box (every sample outside it is 0, and
        // FAST writes no counters); DEBUG/COUNTED need the support box for n_lo/n_hi.
        float t0 = -3.0e38f, t1 = 3.0e38f;
        bool miss = false;
        const float rr = sp.tile_r;
        float lo[3] = {0.0f, 0.0f, 0.0f}, hi[3] = {v.sx1, v.sy1, v.sz1};
        if (!DEBUG && !COUNT) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                lo[q] = sp.alo[q];
                hi[q] = sp.ahi[q];
            }
        }
        slab(c.ox - lo[0] + rr, sp.Dg[0], sp.invD[0], hi[0] - lo[0] + 2.0f * rr, 0.0f, t0, t1, miss);
        slab(c.oy - lo[1] + rr, sp.Dg[1], sp.invD[1], hi[1] - lo[1] + 2.0f * rr, 0.0f, t0, t1, miss);
        slab(c.oz - lo[2] + rr, sp.Dg[2], sp.invD[2], hi[2] - lo[2] + 2.0f * rr, 0.0f, t0, t1, miss);
        if (miss || !(t0 <= t1) || t1 < 0.0f) {
            if (valid) {
                out_rgbt[o] = make_float4(0.0f, 0.0f, 0.0f, 1.0f);
                out_depth[o] = 0.0f;
                if (DEBUG) {
                    uint32_t* dbg = out_debug + o * 6;
                    dbg[0] = dbg[1] = dbg[2] = dbg[3] = dbg[4] = dbg[5] = 0u;
                }
            }
            return;   // uniform over the CTA
        }
    }
#if NSL_STAGE
    {
        const uint4* src = reinterpret_cast<const uint4*>(sp.occ);
        const int n4 = sp.occ_words >> 2;
        for (int i = threadIdx.x; i < n4; i += blockDim.x) smask4[i] = __ldg(src + i);
    }
    __syncthreads();
#endif
    if (!COUNT && !valid) return;

    uint32_t c_prim = 0, c_light = 0, c_gath = 0, c_occ = 0, c_tp = 0, c_tl = 0;
    if (valid) {
        // ---- a2: ray (C3), jitter (C4)
        Ray r;
        float P[4];
        float inv[3];
        const float fpx = (float)px, fpy = (float)py;
        if (PROJ == 0) {
            r.ox = __fmaf_rn(fpy, sp.Ey[0], __fmaf_rn(fpx, sp.Ex[0], sp.B[0]));
            r.oy = __fmaf_rn(fpy, sp.Ey[1], __fmaf_rn(fpx, sp.Ex[1], sp.B[1]));
            r.oz = __fmaf_rn(fpy, sp.Ey[2], __fmaf_rn(fpx, sp.Ex[2], sp.B[2]));
            r.dx = sp.Dg[0];
            r.dy = sp.Dg[1];
            r.dz = sp.Dg[2];
            inv[0] = sp.invD[0];
            inv[1] = sp.invD[1];
            inv[2] = sp.invD[2];
#pragma unroll
            for (int l = 0; l < 4; ++l) P[l] = sp.P[l];
        } else {
            const float d0 = __fmaf_rn(fpy, sp.Ey[0], __fmaf_rn(fpx, sp.Ex[0], sp.F0[0]));
            const float d1 = __fmaf_rn(fpy, sp.Ey[1], __fmaf_rn(fpx, sp.Ex[1], sp.F0[1]));
            const float d2 = __fmaf_rn(fpy, sp.Ey[2], __fmaf_rn(fpx, sp.Ex[2], sp.F0[2]));
            const float q = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)));
            const float iq = __fdiv_rn(1.0f, __fsqrt_rn(q));
            const float dir0 = __fmul_rn(d0, iq), dir1 = __fmul_rn(d1, iq), dir2 = __fmul_rn(d2, iq);
            r.dx = __fmul_rn(dir0, sp.inv_dx);
            r.dy = __fmul_rn(dir1, sp.inv_dx);
            r.dz = __fmul_rn(dir2, sp.inv_dx);
            r.ox = sp.Oe[0];
            r.oy = sp.Oe[1];
            r.oz = sp.Oe[2];
            inv[0] = r.dx != 0.0f ? 1.0f / r.dx : 0.0f;
            inv[1] = r.dy != 0.0f ? 1.0f / r.dy : 0.0f;
            inv[2] = r.dz != 0.0f ? 1.0f / r.dz : 0.0f;
#pragma unroll
            for (int l = 0; l < 4; ++l)
                P[l] = hg32(mc.g, sp.Ln[l][0] * dir0 + sp.Ln[l][1] * dir1 + sp.Ln[l][2] * dir2);
        }
        r.h = mc.h;
        const uint32_t pix = (uint32_t)py * (uint32_t)W + (uint32_t)px;
        r.delta = mc.jitter ? jitter_delta(jitter_hash(mc.seed_lo, mc.seed_hi, sp.frame_id, pix), mc.h) : 0.0f;

        // ---- C5: the steps actually marched are the in-support steps of [1, N] whose
        //      positions lie in the occupied box (every other sample is exactly 0).
        //      FAST: bracket the box's step range (float slab test, +-1 step) and make
        //      its two ends exact with prescribed-op support tests (the in-support set
        //      is contiguous, so the whole range is then in support).  DEBUG/COUNTED
        //      also need the exact support range n_lo..n_hi for the bookkeeping.
        int n_lo = 0, n_hi = -1;
        const float inv_h = 1.0f / mc.h;
        if (DEBUG || COUNT) clip_ray(r, v, inv, inv_h, mc.Ncap, n_lo, n_hi);
        int m_lo, m_hi;
        {
            float u0 = -3.0e38f, u1 = 3.0e38f;
            bool miss = false;
            slab(r.ox - sp.alo[0], r.dx, inv[0], sp.ahi[0] - sp.alo[0], 1e-3f, u0, u1, miss);
            slab(r.oy - sp.alo[1], r.dy, inv[1], sp.ahi[1] - sp.alo[1], 1e-3f, u0, u1, miss);
            slab(r.oz - sp.alo[2], r.dz, inv[2], sp.ahi[2] - sp.alo[2], 1e-3f, u0, u1, miss);
            if (miss || !(u0 <= u1)) {
                m_lo = 1;
                m_hi = 0;
            } else if (DEBUG || COUNT) {
                m_lo = n_lo;
                m_hi = n_hi;
                const float a = floorf((u0 - r.delta) * inv_h) - 1.0f, b = ceilf((u1 - r.delta) * inv_h) + 1.0f;
                if (a > (float)m_lo) m_lo = a < (float)m_hi ? (int)a : m_hi + 1;
                if (b < (float)m_hi) m_hi = b > (float)m_lo ? (int)b : m_lo - 1;
            } else {
                const float a = fmaxf(floorf((u0 - r.delta) * inv_h) - 1.0f, 1.0f);
                const float b = fminf(ceilf((u1 - r.delta) * inv_h) + 1.0f, (float)mc.Ncap);
                if (a <= b) {
                    m_lo = (int)a;
                    m_hi = (int)b;
                    while (m_lo <= m_hi && !r.in(v, m_lo)) ++m_lo;
                    while (m_hi >= m_lo && !r.in(v, m_hi)) --m_hi;
                } else {
                    m_lo = 1;
                    m_hi = 0;
                }
            }
        }

        // ---- a4-a7 march
        float tau = 0.0f, T = 1.0f, Dout = 0.0f;
        float S[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        int n_hit = 0, n_term = n_hi > 0 ? n_hi : 0;
        uint32_t n_occ = 0, lsamp = 0;
        // C9 precondition per ray: step 1 lies outside the support (i.e. n_lo >= 2)
        const bool front_fast = !DEBUG && PROJ == 0 && sp.front_ok && m_lo <= m_hi && !r.in(v, 1);
        const bool paired = sp.pair12 != 0;
        float nf = (float)m_lo;
        for (int n = m_lo; n <= m_hi; ++n, nf += 1.0f) {
            float t, x, y, z;
            r.atf(nf, t, x, y, z);
            if (COUNT) ++c_tp;
            const float rho = sample<LAYOUT, COUNT>(v, x, y, z, c_gath);
            if (rho > 0.0f) {
                ++n_occ;
                const float sig_t = mc.kappa * rho;
                const float sig_s = mc.alpha * sig_t;
                if (n_hit == 0 && sig_s > mc.tau_d) {   // C6
                    n_hit = n;
                    Dout = t;
                }
                const float s = sig_t * mc.h;            // C7
                const float Tp = T;
                tau += s;
                T = __expf(-tau);
                float A;
                if (mc.form == NSL_OPACITY_EXP) A = mc.alpha * (Tp - T);
                else if (mc.form == NSL_OPACITY_RIEMANN) A = mc.alpha * Tp * s;
                else A = Tp * sig_s;
                const float kl = mc.hl * mc.kappa;
                if (paired) {                              // C8: top/bottom in one loop
                    int Ma, Mb, ma, mb;
                    if (DEBUG || COUNT) {
                        Ma = light_count(v, x, y, z, sp.Lg[1][0], sp.Lg[1][1], sp.Lg[1][2], mc.hl, sp.lim[1], sp.ilh[1]);
                        Mb = light_count(v, x, y, z, sp.Lg[2][0], sp.Lg[2][1], sp.Lg[2][2], mc.hl, sp.lim[2], sp.ilh[2]);
                        float ra[3], rb[3];
                        march_region(sp, v, 1, z, ra);
                        march_region(sp, v, 2, z, rb);
                        ma = min(Ma, box_count(x, y, z, ra, sp.ilh[1]));
                        mb = min(Mb, box_count(x, y, z, rb, sp.ilh[2]));
                    } else {
                        Ma = Mb = 0;
                        float ra[3], rb[3];
                        march_region(sp, v, 1, z, ra);
                        march_region(sp, v, 2, z, rb);
                        ma = light_bound(v, x, y, z, sp.Lg[1][0], sp.Lg[1][1], sp.Lg[1][2], mc.hl, sp.lim[1], sp.ilh[1], ra);
                        mb = light_bound(v, x, y, z, sp.Lg[2][0], sp.Lg[2][1], sp.Lg[2][2], mc.hl, sp.lim[2], sp.ilh[2], rb);
                    }
                    if (COUNT) c_tl += (uint32_t)(ma + mb);
                    float sa, sb;
                    light_sum_pair<LAYOUT, COUNT>(v, x, y, z, sp.Lg[1][0], sp.Lg[1][1], sp.Lg[1][2], mc.hl, ma, mb, sa,
                                                  sb, c_gath);
                    S[1] = __fmaf_rn(A, __expf(-kl * sa), S[1]);
                    S[2] = __fmaf_rn(A, __expf(-kl * sb), S[2]);
                    lsamp += (uint32_t)(Ma + Mb);
                }
#pragma unroll
                for (int l = 0; l < 4; ++l) {             // C8 + C10
                    if (l < mc.n_lights && !(paired && (l == 1 || l == 2))) {
                        float Tl;
                        const float lx = sp.Lg[l][0], ly = sp.Lg[l][1], lz = sp.Lg[l][2];
                        if (l == 0 && front_fast) {
                            Tl = Tp;                      // C9: T^front_n = T_{n-1}
                            if (COUNT) lsamp += (uint32_t)light_count(v, x, y, z, lx, ly, lz, mc.hl, sp.lim[l], sp.ilh[l]);
                        } else {
                            int M, mm;
                            if (DEBUG || COUNT) {
                                M = light_count(v, x, y, z, lx, ly, lz, mc.hl, sp.lim[l], sp.ilh[l]);
                                float rl[3];
                                march_region(sp, v, l, z, rl);
                                mm = min(M, box_count(x, y, z, rl, sp.ilh[l]));
                            } else {
                                M = 0;
                                float rl[3];
                                march_region(sp, v, l, z, rl);
                                mm = light_bound(v, x, y, z, lx, ly, lz, mc.hl, sp.lim[l], sp.ilh[l], rl);
                            }
                            if (COUNT) c_tl += (uint32_t)mm;
                            const float sum = light_sum<LAYOUT, COUNT>(v, x, y, z, lx, ly, lz, mc.hl, mm, c_gath);
                            Tl = __expf(-kl * sum);
                            lsamp += (uint32_t)M;
                        }
                        S[l] = __fmaf_rn(A, Tl, S[l]);
                    }
                }
                if (T < mc.t_min) {                       // C11
                    n_term = n;
                    break;
                }
            }
        }
        // ---- a6/a8: L_c = sum_l rgb_lc P_l S_l; vectorised stores
        float L0 = 0.0f, L1 = 0.0f, L2 = 0.0f;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            if (l < mc.n_lights) {
                const float w = P[l] * S[l];
                L0 += sp.rgb[l][0] * w;
                L1 += sp.rgb[l][1] * w;
                L2 += sp.rgb[l][2] * w;
            }
        }
        out_rgbt[o] = make_float4(L0, L1, L2, T);
        out_depth[o] = Dout;
        const bool hit_support = n_lo > 0 && n_hi >= n_lo;
        if (DEBUG) {
            uint32_t* dbg = out_debug + o * 6;
            dbg[0] = hit_support ? (uint32_t)n_lo : 0u;
            dbg[1] = hit_support ? (uint32_t)n_hi : 0u;
            dbg[2] = (uint32_t)n_hit;
            dbg[3] = (uint32_t)n_term;
            dbg[4] = n_occ;
            dbg[5] = lsamp;
        }
        if (COUNT) {
            c_prim = hit_support ? (uint32_t)(n_term - n_lo + 1) : 0u;
            c_light = lsamp;
            c_occ = n_occ;
        }
    }
    if (COUNT) {
        __shared__ unsigned int red[6];
        if (threadIdx.x < 6) red[threadIdx.x] = 0;
        __syncthreads();
        atomicAdd(&red[0], c_prim);
        atomicAdd(&red[1], c_light);
        atomicAdd(&red[2], c_gath);
        atomicAdd(&red[3], c_occ);
        atomicAdd(&red[4], c_tp);
        atomicAdd(&red[5], c_tl);
        __syncthreads();
        if (threadIdx.x < 6) atomicAdd(counters + threadIdx.x, (unsigned long long)red[threadIdx.x]);
    }
}

__global__ void jitter_debug_kernel(MarchConst mc, uint32_t frame, int n, uint32_t* hash, float* delta) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    uint32_t h = jitter_hash(mc.seed_lo, mc.seed_hi, frame, (uint32_t)p);
    hash[p] = h;
    delta[p] = mc.jitter ? jitter_delta(h, mc.h) : 0.0f;
}

template <int LAYOUT, int PROJ, int MODE>
cudaError_t launch_lpm(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, size_t smem, float4* rgbt,
                       float* depth, uint32_t* debug, unsigned long long* counters, const uint32_t* tile_order,
                       cudaStream_t s) {
    const int tiles_x = (W + kTileW - 1) / kTileW, tiles_y = (H + kTileH - 1) / kTileH;
    dim3 grid((unsigned)(tiles_x * tiles_y) * (unsigned)F);
    auto k = march_kernel<LAYOUT, PROJ, MODE>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<grid, kThreads, smem, s>>>(fp, mc, rgbt, depth, debug, counters, W, H, tile_order, F);
    return cudaGetLastError();
}

template <int LAYOUT, int PROJ>
cudaError_t launch_lp(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, size_t smem, float4* rgbt,
                      float* depth, uint32_t* debug, unsigned long long* counters, const uint32_t* to, cudaStream_t s) {
    if (debug) return launch_lpm<LAYOUT, PROJ, kDebug>(fp, mc, F, W, H, smem, rgbt, depth, debug, counters, to, s);
    if (counters) return launch_lpm<LAYOUT, PROJ, kCounted>(fp, mc, F, W, H, smem, rgbt, depth, debug, counters, to, s);
    return launch_lpm<LAYOUT, PROJ, kFast>(fp, mc, F, W, H, smem, rgbt, depth, debug, counters, to, s);
}

template <int LAYOUT>
cudaError_t launch_l(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, int proj, size_t smem,
                     float4* rgbt, float* depth, uint32_t* debug, unsigned long long* counters, const uint32_t* to,
                     cudaStream_t s) {
    return proj == 0 ? launch_lp<LAYOUT, 0>(fp, mc, F, W, H, smem, rgbt, depth, debug, counters, to, s)
                     : launch_lp<LAYOUT, 1>(fp, mc, F, W, H, smem, rgbt, depth, debug, counters, to, s);
}

}  // namespace

int march_tile_w() { return kTileW; }
int march_tile_h() { return kTileH; }

cudaError_t launch_march(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, int projection, int layout,
                         int max_occ_words, float4* rgbt, float* depth, uint32_t* debug,
                         unsigned long long* counters, const uint32_t* tile_order, cudaStream_t s) {
    const size_t smem = NSL_STAGE ? sizeof(FrameParams) + (size_t)max_occ_words * 4 : 0;
    switch (layout) {
        case kLinearF32:
            return launch_l<kLinearF32>(fp, mc, F, W, H, projection, smem, rgbt, depth, debug, counters, tile_order, s);
        case kQuadF32:
            return launch_l<kQuadF32>(fp, mc, F, W, H, projection, smem, rgbt, depth, debug, counters, tile_order, s);
        case kCornerF16:
            return launch_l<kCornerF16>(fp, mc, F, W, H, projection, smem, rgbt, depth, debug, counters, tile_order, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_jitter_debug(const MarchConst& mc, uint32_t frame_id, int n, uint32_t* hash, float* delta,
                                cudaStream_t s) {
    jitter_debug_kernel<<<(n + 255) / 256, 256, 0, s>>>(mc, frame_id, n, hash, delta);
    return cudaGetLastError();
}

}  // namespace nsl
