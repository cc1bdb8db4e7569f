// bake.cu — NEXT-1: reference single-scatter six-way bake (DESIGN.md §10,
// B1-B6): the six-way lightmaps {L_x^±, L_y^±, L_z^±},
// transparency and an emissive carrier packed as the two RGBA textures of
// Fig. 2 (L255), by jittered fixed-step quadrature of the single-scatter
// integral ("single bounce ... g = 0 ... samples per pixel", L477).
//
// One pixel per 16 lanes: lane l takes samples s = l, l+16, ... (in order) and
// a fixed shuffle tree sums the 16 partials, so the result is deterministic and
// independent of scheduling.  The lanes of a pixel trace sub-pixel-jittered
// rays through the same voxels, so their gathers coalesce far better than the
// guiding map's per-pixel-jittered warps.  Sampler, occupancy skip and exact
// support tests are the march's (sampler.cuh).
#include "sampler.cuh"

namespace nsl {
namespace {

constexpr int kBakeThreads = 128;          // 8 pixels (4 x 2) x 16 sample lanes
constexpr int kBakeTileW = 4, kBakeTileH = 2;

// B2: counter-based stream keyed by (seed, frame, pixel, sample)
__device__ __forceinline__ void bake_random(uint32_t seed_lo, uint32_t seed_hi, uint32_t frame, uint32_t pixel,
                                            uint32_t sample, float u[4]) {
    uint32_t h = fmix32(seed_lo ^ 0x85EBCA6Bu);
    h = fmix32(h ^ seed_hi);
    h = fmix32(h ^ frame);
    h = fmix32(h ^ pixel);
    h = fmix32(h ^ sample);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        u[i] = __fmul_rn(__uint2float_rn(h >> 8), 5.9604644775390625e-08f);
        h = fmix32(h + 0x9E3779B9u);
    }
}

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double norm3d(const double a[3]) {
    return __dsqrt_rn(da(da(dm(a[0], a[0]), dm(a[1], a[1])), dm(a[2], a[2])));
}
__device__ __forceinline__ void cross3d(const double a[3], const double b[3], double o[3]) {
    o[0] = ds(dm(a[1], b[2]), dm(a[2], b[1]));
    o[1] = ds(dm(a[2], b[0]), dm(a[0], b[2]));
    o[2] = ds(dm(a[0], b[1]), dm(a[1], b[0]));
}

// B1: the six billboard-axis lights per frame (fp64, C3's basis operations),
// plus the estimate helpers of the march (exit planes, 1/(L h_bl), occupied box).
__global__ void bake_setup_kernel(const FrameIn* __restrict__ in, const FrameParams* __restrict__ fps, int F,
                                  float hbl, float g, BakeFrame* __restrict__ out) {
    const int fi = blockIdx.x * blockDim.x + threadIdx.x;
    if (fi >= F) return;
    const nsl_camera& cam = in[fi].cam;
    const FrameParams& sp = fps[fi];
    const double dx = (double)in[fi].vol.dx;
    double Fw[3] = {cam.forward[0], cam.forward[1], cam.forward[2]};
    double Up[3] = {cam.up[0], cam.up[1], cam.up[2]};
    const double nf = norm3d(Fw);
    double f[3] = {dd(Fw[0], nf), dd(Fw[1], nf), dd(Fw[2], nf)};
    double c[3];
    cross3d(f, Up, c);
    const double nc = norm3d(c);
    double r[3] = {dd(c[0], nc), dd(c[1], nc), dd(c[2], nc)};
    double u[3];
    cross3d(r, f, u);
    double n[6][3];
    for (int a = 0; a < 3; ++a) {
        n[0][a] = r[a];
        n[1][a] = u[a];
        n[2][a] = f[a];
        n[3][a] = -r[a];
        n[4][a] = -u[a];
        n[5][a] = -f[a];
    }
    BakeFrame b;
    b.lz0 = 0;
    for (int l = 0; l < 6; ++l) {
        for (int a = 0; a < 3; ++a) {
            b.Ln[l][a] = (float)n[l][a];
            b.Lg[l][a] = (float)dd(n[l][a], dx);
        }
        // phase for orthographic cameras (dir = fwd): HG(g, Ln . fwd) from the fp32 vectors
        const double cth = ((double)b.Ln[l][0] * sp.fwd[0] + (double)b.Ln[l][1] * sp.fwd[1]) +
                           (double)b.Ln[l][2] * sp.fwd[2];
        const double dg = (1.0 + (double)g * g) - 2.0 * (double)g * cth;
        b.P[l] = (float)((1.0 - (double)g * g) / ((4.0 * 3.141592653589793) * (dg * sqrt(dg))));
        for (int a = 0; a < 3; ++a) {
            const float L = b.Lg[l][a];
            b.lim[l][a] = L > 0.0f ? sp.supp[a] : (L < 0.0f ? 0.0f : 3.0e38f);
            b.alim[l][a] = L > 0.0f ? sp.ahi[a] : (L < 0.0f ? sp.alo[a] : 3.0e38f);
            b.ilh[l][a] = L != 0.0f ? 1.0f / (L * hbl) : 1.0f;
        }
        if (b.Lg[l][2] == 0.0f) b.lz0 |= 1 << l;
    }
    out[fi] = b;
}

// Number of leading light samples (B4, jittered offset o3 = u3 h_bl) that can be
// nonzero: estimate of the region count (+1 slack; the region lies inside the
// support, so its estimate never exceeds the support's), then shrunk with exact
// prescribed-op support tests.
__device__ __forceinline__ int bake_light_bound(const Vol& v, float ux, float uy, float uz, float lx, float ly,
                                                float lz, float hbl, float o3, float u3, const float ilh[3],
                                                const float reg[3]) {
    const float mr = fminf(fminf((reg[0] - ux) * ilh[0], (reg[1] - uy) * ilh[1]), (reg[2] - uz) * ilh[2]);
    float m = floorf(mr - u3) + 2.0f;
    m = fminf(fmaxf(m, 0.0f), 16777216.0f);
    while (m > 0.0f) {
        const float s = __fmaf_rn(m - 1.0f, hbl, o3);
        if (inside(v, __fmaf_rn(s, lx, ux), __fmaf_rn(s, ly, uy), __fmaf_rn(s, lz, uz))) break;
        m -= 1.0f;
    }
    return (int)m;
}

// region exit planes for light l from height uz (slab box for horizontal lights)
__device__ __forceinline__ void bake_region(const FrameParams& sp, const BakeFrame& bf, const Vol& v, int l, float uz,
                                            float out[3]) {
    if ((bf.lz0 >> l) & 1) {
        const int iz = __float_as_int(__fadd_rd(uz, kFloorBias)) - 0x4B400000;
        const int bz = iz >> v.shift;
        const int* slab = reinterpret_cast<const int*>(v.occ) + sp.slab_off;
        const int2 mn = __ldg(reinterpret_cast<const int2*>(slab + 2 * bz));
        const int2 mx = __ldg(reinterpret_cast<const int2*>(slab + 2 * sp.occ_nbz + 2 * bz));
        const float B = (float)(1 << v.shift);
        const float lox = (float)mn.x * B, hix = fminf((float)(mx.x + 1) * B, v.sx1);
        const float loy = (float)mn.y * B, hiy = fminf((float)(mx.y + 1) * B, v.sy1);
        const float Lx = bf.Lg[l][0], Ly = bf.Lg[l][1];
        out[0] = Lx > 0.0f ? hix : (Lx < 0.0f ? lox : 3.0e38f);
        out[1] = Ly > 0.0f ? hiy : (Ly < 0.0f ? loy : 3.0e38f);
        out[2] = 3.0e38f;
    } else {
        out[0] = bf.alim[l][0];
        out[1] = bf.alim[l][1];
        out[2] = bf.alim[l][2];
    }
}

#ifndef NSL_BAKE_MINB
#define NSL_BAKE_MINB 12  // min resident CTAs per SM (register cap 40: 48 warps/SM); measured 1 -> 14.3, 8 -> 11.1,
                          // 12 -> 10.1, 14/16 -> 12.6 ms per C2 frame (spills)
#endif
template <int LAYOUT, int PROJ>
__global__ void __launch_bounds__(kBakeThreads, NSL_BAKE_MINB) bake_kernel(const FrameParams* __restrict__ fps,
                                                          const BakeFrame* __restrict__ bfs, const BakeConst bc,
                                                          float4* __restrict__ out, int W, int H, int tiles_x) {
    const int f = blockIdx.y;
    const FrameParams& sp = fps[f];
    const BakeFrame& bf = bfs[f];
    const int lane16 = threadIdx.x & 15, slot = threadIdx.x >> 4;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int px = tx * kBakeTileW + (slot & 3), py = ty * kBakeTileH + (slot >> 2);
    const bool valid = px < W && py < H;

    Vol v;
    v.data = sp.data;
    v.occ = sp.occ;
    v.sy = sp.sy;
    v.sz = sp.sz;
    v.shift = sp.occ_shift;
    v.nbx = sp.occ_nbx;
    v.nby = sp.occ_nby;
    v.sx1 = sp.supp[0];
    v.sy1 = sp.supp[1];
    v.sz1 = sp.supp[2];
    v.mask_words = sp.slab_off;

    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t gath = 0;
    const uint32_t pix = (uint32_t)py * (uint32_t)W + (uint32_t)px;
    const float hb = bc.hb, hbl = bc.hbl, inv_hb = 1.0f / bc.hb;
    for (int s = lane16; valid && s < bc.spp; s += 16) {
        float u4[4];
        bake_random(bc.seed_lo, bc.seed_hi, sp.frame_id, pix, (uint32_t)s, u4);
        const float fx = __fadd_rn((float)px, __fsub_rn(u4[0], 0.5f));
        const float fy = __fadd_rn((float)py, __fsub_rn(u4[1], 0.5f));
        Ray r;
        float inv[3], P[6];
        if (PROJ == 0) {
            r.ox = __fmaf_rn(fy, sp.Ey[0], __fmaf_rn(fx, sp.Ex[0], sp.B[0]));
            r.oy = __fmaf_rn(fy, sp.Ey[1], __fmaf_rn(fx, sp.Ex[1], sp.B[1]));
            r.oz = __fmaf_rn(fy, sp.Ey[2], __fmaf_rn(fx, sp.Ex[2], sp.B[2]));
            r.dx = sp.Dg[0];
            r.dy = sp.Dg[1];
            r.dz = sp.Dg[2];
            inv[0] = sp.invD[0];
            inv[1] = sp.invD[1];
            inv[2] = sp.invD[2];
#pragma unroll
            for (int l = 0; l < 6; ++l) P[l] = bf.P[l];
        } else {
            const float d0 = __fmaf_rn(fy, sp.Ey[0], __fmaf_rn(fx, sp.Ex[0], sp.F0[0]));
            const float d1 = __fmaf_rn(fy, sp.Ey[1], __fmaf_rn(fx, sp.Ex[1], sp.F0[1]));
            const float d2 = __fmaf_rn(fy, sp.Ey[2], __fmaf_rn(fx, sp.Ex[2], sp.F0[2]));
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
            for (int l = 0; l < 6; ++l) {
                const float cth = bf.Ln[l][0] * dir0 + bf.Ln[l][1] * dir1 + bf.Ln[l][2] * dir2;
                const float dg = (1.0f + bc.g * bc.g) - 2.0f * bc.g * cth;
                P[l] = (1.0f - bc.g * bc.g) / (12.566370614359172f * dg * sqrtf(dg));
            }
        }
        const float o2 = __fmul_rn(u4[2], hb), o3 = __fmul_rn(u4[3], hbl);
        r.h = hb;
        r.delta = o2;
        // B3 steps k >= 0 inside the occupied box (bracket) and the support (exact ends)
        int k0, k1;
        {
            float t0 = -3.0e38f, t1 = 3.0e38f;
            bool miss = false;
            slab(r.ox - sp.alo[0], r.dx, inv[0], sp.ahi[0] - sp.alo[0], 1e-3f, t0, t1, miss);
            slab(r.oy - sp.alo[1], r.dy, inv[1], sp.ahi[1] - sp.alo[1], 1e-3f, t0, t1, miss);
            slab(r.oz - sp.alo[2], r.dz, inv[2], sp.ahi[2] - sp.alo[2], 1e-3f, t0, t1, miss);
            k0 = 0;
            k1 = -1;
            if (!miss && t0 <= t1) {
                const float a = fmaxf(floorf((t0 - o2) * inv_hb) - 1.0f, 0.0f);
                const float b = fminf(ceilf((t1 - o2) * inv_hb) + 1.0f, (float)bc.Ncap);
                if (a <= b) {
                    k0 = (int)a;
                    k1 = (int)b;
                    while (k0 <= k1 && !r.in(v, k0)) ++k0;
                    while (k1 >= k0 && !r.in(v, k1)) --k1;
                }
            }
        }
        float tau = 0.0f, sc[6] = {0, 0, 0, 0, 0, 0}, em = 0.0f;
        float kf = (float)k0;
        for (int k = k0; k <= k1; ++k, kf += 1.0f) {
            float t, x, y, z;
            r.atf(kf, t, x, y, z);
            const float rho = sample<LAYOUT, true>(v, x, y, z, gath);
            if (!(rho > 0.0f)) continue;
            const float sig_t = bc.kappa * rho;
            const float Tk = __expf(-tau);
            const float w = bc.alpha * sig_t * hb * Tk;          // sigma_s h T_k
            em += (1.0f - bc.alpha) * sig_t * hb * Tk;           // sigma_a h T_k
#pragma unroll
            for (int l = 0; l < 6; ++l) {
                const float lx = bf.Lg[l][0], ly = bf.Lg[l][1], lz = bf.Lg[l][2];
                float reg[3];
                bake_region(sp, bf, v, l, z, reg);
                const int m = bake_light_bound(v, x, y, z, lx, ly, lz, hbl, o3, u4[3], bf.ilh[l], reg);
                float sum = 0.0f;
                float jf = 0.0f;
                for (int j = 1; j <= m; ++j, jf += 1.0f) {
                    const float sj = __fmaf_rn(jf, hbl, o3);
                    sum += sample<LAYOUT, true>(v, __fmaf_rn(sj, lx, x), __fmaf_rn(sj, ly, y), __fmaf_rn(sj, lz, z), gath);
                }
                sc[l] = __fmaf_rn(w * __expf(-(hbl * bc.kappa) * sum), P[l], sc[l]);
            }
            tau += sig_t * hb;
            if (bc.t_min > 0.0f && __expf(-tau) < bc.t_min) break;
        }
        // B6 packing: (right, top, back, T) (left, bottom, front, E)
        acc[0] += sc[0];
        acc[1] += sc[1];
        acc[2] += sc[2];
        acc[3] += __expf(-tau);
        acc[4] += sc[3];
        acc[5] += sc[4];
        acc[6] += sc[5];
        acc[7] += em;
    }
    // deterministic tree over the 16 sample lanes of each pixel
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    if (valid && lane16 == 0) {
        const float inv_spp = 1.0f / (float)bc.spp;
        const size_t o = ((size_t)f * (size_t)W * (size_t)H + pix) * 2;
        out[o] = make_float4(acc[0] * inv_spp, acc[1] * inv_spp, acc[2] * inv_spp, acc[3] * inv_spp);
        out[o + 1] = make_float4(acc[4] * inv_spp, acc[5] * inv_spp, acc[6] * inv_spp, acc[7] * inv_spp);
    }
    if (bc.counters) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) gath += __shfl_xor_sync(0xffffffffu, gath, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(bc.counters, (unsigned long long)gath);
    }
}

template <int LAYOUT>
cudaError_t launch_bake_l(const FrameParams* fp, const BakeFrame* bf, const BakeConst& bc, int F, int W, int H,
                          int proj, float4* out, cudaStream_t s) {
    const int tiles_x = (W + kBakeTileW - 1) / kBakeTileW, tiles_y = (H + kBakeTileH - 1) / kBakeTileH;
    dim3 grid((unsigned)(tiles_x * tiles_y), (unsigned)F);
    if (proj == 0)
        bake_kernel<LAYOUT, 0><<<grid, kBakeThreads, 0, s>>>(fp, bf, bc, out, W, H, tiles_x);
    else
        bake_kernel<LAYOUT, 1><<<grid, kBakeThreads, 0, s>>>(fp, bf, bc, out, W, H, tiles_x);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_bake_setup(const FrameIn* in, const FrameParams* fps, int F, float hbl, float g, BakeFrame* out,
                              cudaStream_t s) {
    bake_setup_kernel<<<(F + 63) / 64, 64, 0, s>>>(in, fps, F, hbl, g, out);
    return cudaGetLastError();
}

cudaError_t launch_bake(const FrameParams* fp, const BakeFrame* bf, const BakeConst& bc, int F, int W, int H,
                        int projection, int layout, float4* out, cudaStream_t s) {
    switch (layout) {
        case kLinearF32: return launch_bake_l<kLinearF32>(fp, bf, bc, F, W, H, projection, out, s);
        case kQuadF32: return launch_bake_l<kQuadF32>(fp, bf, bc, F, W, H, projection, out, s);
        case kCornerF16: return launch_bake_l<kCornerF16>(fp, bf, bc, F, W, H, projection, out, s);
        case kOctF32: return launch_bake_l<kOctF32>(fp, bf, bc, F, W, H, projection, out, s);
        case kBrickOctF32: return launch_bake_l<kBrickOctF32>(fp, bf, bc, F, W, H, projection, out, s);
        case kTex3dF32: return launch_bake_l<kTex3dF32>(fp, bf, bc, F, W, H, projection, out, s);
        case kMortonOctF32: return launch_bake_l<kMortonOctF32>(fp, bf, bc, F, W, H, projection, out, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace nsl
