// march.cu — rows a2, a4-a8: the guiding-map ray march (Algorithm 1,
// L394-407; C3-C12) for sm_100a.
//
// One thread per pixel; a warp marches a coherent 8x4 pixel tile, a CTA a
// 16x8 tile; blockIdx.y is the frame of the batch (row a9).  Sample
// positions use only explicitly rounded fp32 operations (__fmaf_rn,
// __fmul_rn) so that every index decision is bit-identical to the oracle
// (C14); values are fp32 with FMA lerps.  The step range is
// clipped exactly (C5) and each light march's length is computed exactly
// (C8) so the inner loops carry no bounds tests.
#include <cuda_fp16.h>

#include "nsl_internal.cuh"

namespace nsl {
namespace {

constexpr int kTileW = 16, kTileH = 8, kThreads = 128;

struct Vol {
    const void* __restrict__ data;
    int sy, sz;
    float sx1, sy1, sz1;   // support upper bounds n+1
};

__device__ __forceinline__ float lerpf(float a, float b, float t) { return __fmaf_rn(t, b - a, a); }

__device__ __forceinline__ bool inside(const Vol& v, float x, float y, float z) {
    return x > 0.0f && x < v.sx1 && y > 0.0f && y < v.sy1 && z > 0.0f && z < v.sz1;
}

// C1 trilinear at an in-support padded-index position (corners always exist
// thanks to the apron).  floor and fraction are exact in fp32.
template <int LAYOUT>
__device__ __forceinline__ float sample(const Vol& v, float x, float y, float z) {
    const float fx0 = floorf(x), fy0 = floorf(y), fz0 = floorf(z);
    const float fx = __fsub_rn(x, fx0), fy = __fsub_rn(y, fy0), fz = __fsub_rn(z, fz0);
    const int ix = (int)fx0, iy = (int)fy0, iz = (int)fz0;
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
        const float4 q0 = __ldg(p), q1 = __ldg(p + v.sz);
        const float x00 = lerpf(q0.x, q0.y, fx), x10 = lerpf(q0.z, q0.w, fx);
        const float x01 = lerpf(q1.x, q1.y, fx), x11 = lerpf(q1.z, q1.w, fx);
        return lerpf(lerpf(x00, x10, fy), lerpf(x01, x11, fy), fz);
    } else {
        const uint4 u = __ldg(static_cast<const uint4*>(v.data) + e);
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
        const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&u.z));
        const float2 d = __half22float2(*reinterpret_cast<const __half2*>(&u.w));
        const float x00 = lerpf(a.x, a.y, fx), x10 = lerpf(b.x, b.y, fx);
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
        t = __fmaf_rn((float)n, h, delta);
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

// C5: exact first/last in-support step in [1, Ncap] (0,-1 if none).  A float
// slab test on the box expanded by 1e-3 index units brackets the range to
// within one step; exact per-sample tests then shrink it (the in-support set
// is contiguous because every coordinate is monotone in n).
__device__ __forceinline__ void clip_ray(const Ray& r, const Vol& v, int Ncap, int& n0, int& n1) {
    n0 = 0;
    n1 = -1;
    const float eps = 1e-3f;
    float t0 = -3.0e38f, t1 = 3.0e38f;
    const float o[3] = {r.ox, r.oy, r.oz}, d[3] = {r.dx, r.dy, r.dz}, s[3] = {v.sx1, v.sy1, v.sz1};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (d[a] != 0.0f) {
            const float inv = 1.0f / d[a];
            float ta = (-eps - o[a]) * inv, tb = (s[a] + eps - o[a]) * inv;
            if (ta > tb) {
                const float tt = ta;
                ta = tb;
                tb = tt;
            }
            t0 = fmaxf(t0, ta);
            t1 = fminf(t1, tb);
        } else if (!(o[a] > -eps && o[a] < s[a] + eps)) {
            return;
        }
    }
    if (!(t0 <= t1)) return;
    float a = floorf((t0 - r.delta) / r.h), b = ceilf((t1 - r.delta) / r.h);
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
__device__ __forceinline__ int light_count(const Vol& v, float ux, float uy, float uz, float lx, float ly, float lz,
                                           float hl) {
    float smax = 3.0e38f;
    if (lx > 0.0f) smax = fminf(smax, __fdividef(v.sx1 - ux, lx));
    else if (lx < 0.0f) smax = fminf(smax, __fdividef(-ux, lx));
    if (ly > 0.0f) smax = fminf(smax, __fdividef(v.sy1 - uy, ly));
    else if (ly < 0.0f) smax = fminf(smax, __fdividef(-uy, ly));
    if (lz > 0.0f) smax = fminf(smax, __fdividef(v.sz1 - uz, lz));
    else if (lz < 0.0f) smax = fminf(smax, __fdividef(-uz, lz));
    float mf = floorf(__fdividef(smax, hl));
    mf = fminf(fmaxf(mf, 0.0f), 16777216.0f);
    int M = (int)mf;
    auto in_j = [&](int j) {
        const float s = __fmul_rn((float)j, hl);
        return inside(v, __fmaf_rn(s, lx, ux), __fmaf_rn(s, ly, uy), __fmaf_rn(s, lz, uz));
    };
    while (M > 0 && !in_j(M)) --M;
    while (in_j(M + 1)) ++M;
    return M;
}

// sum of rho over j = 1..M along the light (all in support)
template <int LAYOUT>
__device__ __forceinline__ float light_sum(const Vol& v, float ux, float uy, float uz, float lx, float ly, float lz,
                                           float hl, int M) {
    float acc0 = 0.0f, acc1 = 0.0f;
    int j = 1;
    for (; j + 1 <= M; j += 2) {
        const float s0 = __fmul_rn((float)j, hl), s1 = __fmul_rn((float)(j + 1), hl);
        acc0 += sample<LAYOUT>(v, __fmaf_rn(s0, lx, ux), __fmaf_rn(s0, ly, uy), __fmaf_rn(s0, lz, uz));
        acc1 += sample<LAYOUT>(v, __fmaf_rn(s1, lx, ux), __fmaf_rn(s1, ly, uy), __fmaf_rn(s1, lz, uz));
    }
    if (j <= M) {
        const float s0 = __fmul_rn((float)j, hl);
        acc0 += sample<LAYOUT>(v, __fmaf_rn(s0, lx, ux), __fmaf_rn(s0, ly, uy), __fmaf_rn(s0, lz, uz));
    }
    return acc0 + acc1;
}

__device__ __forceinline__ float hg32(float g, float c) {
    const float d = (1.0f + g * g) - 2.0f * g * c;
    return (1.0f - g * g) / (12.566370614359172f * d * sqrtf(d));
}

template <int LAYOUT, int PROJ, bool DEBUG>
__global__ void __launch_bounds__(kThreads) march_kernel(const FrameParams* __restrict__ fps, const MarchConst mc,
                                                         float4* __restrict__ out_rgbt, float* __restrict__ out_depth,
                                                         uint32_t* __restrict__ out_debug, int W, int H,
                                                         int tiles_x) {
    __shared__ __align__(16) FrameParams sp;
    const int f = blockIdx.y;
    {
        const int4* src = reinterpret_cast<const int4*>(fps + f);
        int4* dst = reinterpret_cast<int4*>(&sp);
        for (int i = threadIdx.x; i < (int)(sizeof(FrameParams) / 16); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int px = tx * kTileW + (warp & 1) * 8 + (lane & 7);
    const int py = ty * kTileH + (warp >> 1) * 4 + (lane >> 3);
    if (px >= W || py >= H) return;

    Vol v;
    v.data = sp.data;
    v.sy = sp.sy;
    v.sz = sp.sz;
    v.sx1 = sp.supp[0];
    v.sy1 = sp.supp[1];
    v.sz1 = sp.supp[2];

    // ---- a2: ray (C3), jitter (C4)
    Ray r;
    float P[4];
    const float fpx = (float)px, fpy = (float)py;
    if (PROJ == 0) {
        r.ox = __fmaf_rn(fpy, sp.Ey[0], __fmaf_rn(fpx, sp.Ex[0], sp.B[0]));
        r.oy = __fmaf_rn(fpy, sp.Ey[1], __fmaf_rn(fpx, sp.Ex[1], sp.B[1]));
        r.oz = __fmaf_rn(fpy, sp.Ey[2], __fmaf_rn(fpx, sp.Ex[2], sp.B[2]));
        r.dx = sp.Dg[0];
        r.dy = sp.Dg[1];
        r.dz = sp.Dg[2];
#pragma unroll
        for (int l = 0; l < 4; ++l) P[l] = sp.P[l];
    } else {
        const float d0 = __fmaf_rn(fpy, sp.Ey[0], __fmaf_rn(fpx, sp.Ex[0], sp.F0[0]));
        const float d1 = __fmaf_rn(fpy, sp.Ey[1], __fmaf_rn(fpx, sp.Ex[1], sp.F0[1]));
        const float d2 = __fmaf_rn(fpy, sp.Ey[2], __fmaf_rn(fpx, sp.Ex[2], sp.F0[2]));
        const float q = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)));
        const float inv = __fdiv_rn(1.0f, __fsqrt_rn(q));
        const float dir0 = __fmul_rn(d0, inv), dir1 = __fmul_rn(d1, inv), dir2 = __fmul_rn(d2, inv);
        r.dx = __fmul_rn(dir0, sp.inv_dx);
        r.dy = __fmul_rn(dir1, sp.inv_dx);
        r.dz = __fmul_rn(dir2, sp.inv_dx);
        r.ox = sp.Oe[0];
        r.oy = sp.Oe[1];
        r.oz = sp.Oe[2];
#pragma unroll
        for (int l = 0; l < 4; ++l) P[l] = hg32(mc.g, sp.Ln[l][0] * dir0 + sp.Ln[l][1] * dir1 + sp.Ln[l][2] * dir2);
    }
    r.h = mc.h;
    const uint32_t pix = (uint32_t)py * (uint32_t)W + (uint32_t)px;
    r.delta = mc.jitter ? jitter_delta(jitter_hash(mc.seed_lo, mc.seed_hi, sp.frame_id, pix), mc.h) : 0.0f;

    // ---- C5 clip
    int n_lo, n_hi;
    clip_ray(r, v, mc.Ncap, n_lo, n_hi);

    // ---- a4-a7 march
    float tau = 0.0f, T = 1.0f, Dout = 0.0f;
    float S[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    int n_hit = 0, n_term = n_hi > 0 ? n_hi : 0;
    uint32_t n_occ = 0, lsamp = 0;
    const bool front_fast = !DEBUG && PROJ == 0 && sp.front_ok && n_lo >= 2;
    for (int n = n_lo; n <= n_hi; ++n) {
        float t, x, y, z;
        r.at(n, t, x, y, z);
        const float rho = sample<LAYOUT>(v, x, y, z);
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
#pragma unroll
            for (int l = 0; l < 4; ++l) {             // C8 + C10
                if (l < mc.n_lights) {
                    float Tl;
                    if (l == 0 && front_fast) {
                        Tl = Tp;                      // C9: T^front_n = T_{n-1}
                    } else {
                        const float lx = sp.Lg[l][0], ly = sp.Lg[l][1], lz = sp.Lg[l][2];
                        const int M = light_count(v, x, y, z, lx, ly, lz, mc.hl);
                        const float sum = light_sum<LAYOUT>(v, x, y, z, lx, ly, lz, mc.hl, M);
                        Tl = __expf(-(mc.hl * mc.kappa) * sum);
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
    const size_t o = (size_t)f * (size_t)W * (size_t)H + pix;
    out_rgbt[o] = make_float4(L0, L1, L2, T);
    out_depth[o] = Dout;
    if (DEBUG) {
        uint32_t* dbg = out_debug + o * 6;
        dbg[0] = n_hi >= n_lo && n_lo > 0 ? (uint32_t)n_lo : 0u;
        dbg[1] = n_hi >= n_lo && n_lo > 0 ? (uint32_t)n_hi : 0u;
        dbg[2] = (uint32_t)n_hit;
        dbg[3] = (uint32_t)n_term;
        dbg[4] = n_occ;
        dbg[5] = lsamp;
    }
}

__global__ void jitter_debug_kernel(MarchConst mc, uint32_t frame, int n, uint32_t* hash, float* delta) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    uint32_t h = jitter_hash(mc.seed_lo, mc.seed_hi, frame, (uint32_t)p);
    hash[p] = h;
    delta[p] = mc.jitter ? jitter_delta(h, mc.h) : 0.0f;
}

template <int LAYOUT, int PROJ>
cudaError_t launch_lp(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, float4* rgbt, float* depth,
                      uint32_t* debug, cudaStream_t s) {
    const int tiles_x = (W + kTileW - 1) / kTileW, tiles_y = (H + kTileH - 1) / kTileH;
    dim3 grid((unsigned)(tiles_x * tiles_y), (unsigned)F);
    if (debug)
        march_kernel<LAYOUT, PROJ, true><<<grid, kThreads, 0, s>>>(fp, mc, rgbt, depth, debug, W, H, tiles_x);
    else
        march_kernel<LAYOUT, PROJ, false><<<grid, kThreads, 0, s>>>(fp, mc, rgbt, depth, debug, W, H, tiles_x);
    return cudaGetLastError();
}

template <int LAYOUT>
cudaError_t launch_l(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, int proj, float4* rgbt,
                     float* depth, uint32_t* debug, cudaStream_t s) {
    return proj == 0 ? launch_lp<LAYOUT, 0>(fp, mc, F, W, H, rgbt, depth, debug, s)
                     : launch_lp<LAYOUT, 1>(fp, mc, F, W, H, rgbt, depth, debug, s);
}

}  // namespace

cudaError_t launch_march(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, int projection, int layout,
                         float4* rgbt, float* depth, uint32_t* debug, cudaStream_t s) {
    switch (layout) {
        case kLinearF32: return launch_l<kLinearF32>(fp, mc, F, W, H, projection, rgbt, depth, debug, s);
        case kQuadF32: return launch_l<kQuadF32>(fp, mc, F, W, H, projection, rgbt, depth, debug, s);
        case kCornerF16: return launch_l<kCornerF16>(fp, mc, F, W, H, projection, rgbt, depth, debug, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_jitter_debug(const MarchConst& mc, uint32_t frame_id, int n, uint32_t* hash, float* delta,
                                cudaStream_t s) {
    jitter_debug_kernel<<<(n + 255) / 256, 256, 0, s>>>(mc, frame_id, n, hash, delta);
    return cudaGetLastError();
}

}  // namespace nsl
