// tv.cu — NEXT-4: the transmittance-volume light model (V2-V5).
//
// tv_setup_kernel: per (frame, lattice slot) the lattice of the light step vector
// d = h_l L_g (V2) in fp64 with explicitly rounded ops, rounded once to fp32, plus the
// sweep window: the lattice range of the occupied box +-2 (every sample outside the
// occupied box is exactly 0, so line sums started at the window are exact, and lookups
// at occupied samples never read outside it).
// tv_sweep_kernel: one thread per lattice line (i, j) of the window; the thread walks
// k over the window once forward (exclusive prefix tau-) and once backward (exclusive
// suffix tau+), sampling the volume through the same occupancy-skipping sampler as
// the march (V3, V4).  Lattice values are float2 (tau+, tau-), i fastest, so a warp's
// stores are coalesced.
#include "sampler.cuh"

namespace nsl {
namespace {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
    return da(da(dm(a[0], b[0]), dm(a[1], b[1])), dm(a[2], b[2]));
}
__device__ __forceinline__ void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = ds(dm(a[1], b[2]), dm(a[2], b[1]));
    o[1] = ds(dm(a[2], b[0]), dm(a[0], b[2]));
    o[2] = ds(dm(a[0], b[1]), dm(a[1], b[0]));
}

// projections of the 8 corners of the box [lo, hi] onto (e1, e2, dhat / ell)
__device__ void box_range(const double lo[3], const double hi[3], const double e1[3], const double e2[3],
                          const double dh[3], double ell, double mn[3], double mx[3]) {
    for (int q = 0; q < 3; ++q) {
        mn[q] = 1e300;
        mx[q] = -1e300;
    }
    for (int c = 0; c < 8; ++c) {
        const double p[3] = {(c & 1) ? hi[0] : lo[0], (c & 2) ? hi[1] : lo[1], (c & 4) ? hi[2] : lo[2]};
        const double v[3] = {dot3(p, e1), dot3(p, e2), dd(dot3(p, dh), ell)};
        for (int q = 0; q < 3; ++q) {
            mn[q] = fmin(mn[q], v[q]);
            mx[q] = fmax(mx[q], v[q]);
        }
    }
}

__global__ void tv_setup_kernel(const FrameParams* __restrict__ fps, int F, int slots, MarchConst mc,
                                TvParams* __restrict__ out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= F * slots) return;
    const int f = idx / slots, slot = idx - f * slots;
    const FrameParams& sp = fps[f];
    const int l = mc.light_mode == NSL_LIGHTS_GUIDE ? 1 : slot;     // the guide pair shares slot 0
    TvParams t;
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = dm((double)mc.hl, (double)sp.Lg[l][a]);
    const double ell = __dsqrt_rn(dot3(d, d));
    double dh[3], c[3], e1[3], e2[3];
    for (int a = 0; a < 3; ++a) dh[a] = dd(d[a], ell);
    const double zh[3] = {0.0, 0.0, 1.0}, xh[3] = {1.0, 0.0, 0.0};
    cross3(dh, zh, c);
    if (__dsqrt_rn(dot3(c, c)) < 1e-6) cross3(dh, xh, c);
    const double nc = __dsqrt_rn(dot3(c, c));
    for (int a = 0; a < 3; ++a) e1[a] = dd(c[a], nc);
    cross3(dh, e1, e2);
    // V2 lattice over the support box
    const double slo[3] = {0.0, 0.0, 0.0}, shi[3] = {sp.supp[0], sp.supp[1], sp.supp[2]};
    double mn[3], mx[3];
    box_range(slo, shi, e1, e2, dh, ell, mn, mx);
    double o0[3];
    int dims[3];
    for (int q = 0; q < 3; ++q) {
        o0[q] = floor(mn[q]) - 1.0;
        dims[q] = (int)(ceil(mx[q]) - o0[q]) + 2;
    }
    // sweep window: the occupied box's range +-2, clamped to the lattice
    const double alo[3] = {sp.alo[0], sp.alo[1], sp.alo[2]}, ahi[3] = {sp.ahi[0], sp.ahi[1], sp.ahi[2]};
    double bmn[3], bmx[3];
    box_range(alo, ahi, e1, e2, dh, ell, bmn, bmx);
    int lo[3], hi[3];
    for (int q = 0; q < 3; ++q) {
        lo[q] = max((int)(floor(bmn[q]) - o0[q]) - 2, 0);
        hi[q] = min((int)(ceil(bmx[q]) - o0[q]) + 2, dims[q] - 1);
    }
    for (int a = 0; a < 3; ++a) {
        t.e1[a] = (float)e1[a];
        t.e2[a] = (float)e2[a];
        t.d[a] = (float)d[a];
        t.dk[a] = (float)dd(dh[a], ell);
    }
    t.a0 = (float)o0[0];
    t.b0 = (float)o0[1];
    t.k0 = (float)o0[2];
    t.kh = mc.kappa * mc.hl;
    t.A = dims[0];
    t.B = dims[1];
    t.K = dims[2];
    t.i_lo = lo[0];
    t.i_hi = hi[0];
    t.j_lo = lo[1];
    t.j_hi = hi[1];
    t.k_lo = lo[2];
    t.k_hi = hi[2];
    t.pad[0] = t.pad[1] = t.pad[2] = 0;
    out[idx] = t;
}

#ifndef NSL_SWEEP_2PASS
#define NSL_SWEEP_2PASS 1
#endif
#ifndef NSL_SWEEP_NOSMEM
#define NSL_SWEEP_NOSMEM 1
#endif
constexpr int kSweepSmemK = 64;   // windows of at most 64 points per line stage in shared memory
template <int LAYOUT>
__global__ void __launch_bounds__(128) tv_sweep_kernel(const FrameParams* __restrict__ fps,
                                                       const TvParams* __restrict__ tvp, int slots, int Astr,
                                                       int Kstr, int64_t slot_elems, int smem_k,
                                                       float2* __restrict__ buf) {
    const int fs = blockIdx.y, f = fs / slots;
    const TvParams& t = tvp[fs];
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = line % Astr, j = line / Astr;
    // the host's stride bounds (capi tv_geometry) hold every device-computed lattice
    NSL_ASSERT(t.A <= Astr && t.K <= Kstr && (int64_t)Astr * t.B * Kstr <= slot_elems);
    if (i < t.i_lo || i > t.i_hi || j < t.j_lo || j > t.j_hi) return;
    const FrameParams& sp = fps[f];
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
    const float af = t.a0 + (float)i, bf = t.b0 + (float)j;
    float base[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) base[a] = __fmaf_rn(bf, t.e2[a], __fmul_rn(af, t.e1[a]));
    float2* col = buf + (int64_t)fs * slot_elems + (int64_t)j * Kstr * Astr + i;
    uint32_t unused = 0;
    auto sample_k = [&](int k) {
        const float kf = t.k0 + (float)k;
        const float x = __fmaf_rn(kf, t.d[0], base[0]), y = __fmaf_rn(kf, t.d[1], base[1]),
                    z = __fmaf_rn(kf, t.d[2], base[2]);
        return t.kh * (inside(v, x, y, z) ? sample<LAYOUT, false>(v, x, y, z, unused) : 0.0f);
    };
    if (t.k_hi - t.k_lo < smem_k) {
        // the line's kappa h rho_k staged in shared memory (a column per thread, conflict-free),
        // then one backward walk writes each lattice point once: tau+ is the exclusive suffix,
        // tau- = total - (tau+ + s_k) (absolute rounding ~ a few ulp of the line total)
        extern __shared__ float sk_s[];
        float* sk = sk_s + threadIdx.x;
        float tot = 0.0f;
        for (int k = t.k_lo; k <= t.k_hi; ++k) {
            const float sv = sample_k(k);
            sk[(k - t.k_lo) * blockDim.x] = sv;
            tot += sv;
        }
        float suf = 0.0f;
        for (int k = t.k_hi; k >= t.k_lo; --k) {
            const float sv = sk[(k - t.k_lo) * blockDim.x];
            col[(int64_t)k * Astr] = make_float2(suf, fmaxf(tot - (suf + sv), 0.0f));
            suf += sv;
        }
        return;
    }
#if NSL_SWEEP_2PASS
    // longer windows: the line total first, then the backward walk re-samples each point
    // (the same values, so the result equals the staged path's) and writes it once
    float tot = 0.0f;
    for (int k = t.k_lo; k <= t.k_hi; ++k) tot += sample_k(k);
    float suf = 0.0f;
    for (int k = t.k_hi; k >= t.k_lo; --k) {
        const float sv = sample_k(k);
        col[(int64_t)k * Astr] = make_float2(suf, fmaxf(tot - (suf + sv), 0.0f));
        suf += sv;
    }
#else
    float acc = 0.0f;                   // V4 tau-: exclusive prefix toward -d
    for (int k = t.k_lo; k <= t.k_hi; ++k) {
        const float sv = sample_k(k);
        col[(int64_t)k * Astr] = make_float2(sv, acc);
        acc += sv;
    }
    acc = 0.0f;                         // V4 tau+: exclusive suffix toward +d
    for (int k = t.k_hi; k >= t.k_lo; --k) {
        float2 e = col[(int64_t)k * Astr];
        const float sv = e.x;
        e.x = acc;
        col[(int64_t)k * Astr] = e;
        acc += sv;
    }
#endif
}

}  // namespace

cudaError_t launch_tv_setup(const FrameParams* fps, int F, int slots, const MarchConst& mc, TvParams* out,
                            cudaStream_t s) {
    const int n = F * slots;
    tv_setup_kernel<<<(n + 63) / 64, 64, 0, s>>>(fps, F, slots, mc, out);
    return cudaGetLastError();
}

cudaError_t launch_tv_sweep(const FrameParams* fps, const TvParams* tvp, int F, int slots, int Astr, int Bstr,
                            int Kstr, const MarchConst& mc, int layout, float2* buf, cudaStream_t s) {
    (void)mc;
    const dim3 grid((unsigned)(((int64_t)Astr * Bstr + 127) / 128), (unsigned)(F * slots));
    const int64_t slot_elems = (int64_t)Astr * Bstr * Kstr;
    // stage up to min(Kstr, 64) points per line: no more shared memory than the longest window
    int smem_k = Kstr < kSweepSmemK ? Kstr : kSweepSmemK;
    if (NSL_SWEEP_2PASS && Kstr > kSweepSmemK * NSL_SWEEP_NOSMEM) smem_k = 0;   // every window may be long
    const size_t smem = (size_t)smem_k * 128 * sizeof(float);
    switch (layout) {
        case kLinearF32: tv_sweep_kernel<kLinearF32><<<grid, 128, smem, s>>>(fps, tvp, slots, Astr, Kstr, slot_elems, smem_k, buf); break;
        case kQuadF32: tv_sweep_kernel<kQuadF32><<<grid, 128, smem, s>>>(fps, tvp, slots, Astr, Kstr, slot_elems, smem_k, buf); break;
        case kCornerF16: tv_sweep_kernel<kCornerF16><<<grid, 128, smem, s>>>(fps, tvp, slots, Astr, Kstr, slot_elems, smem_k, buf); break;
        case kOctF32: tv_sweep_kernel<kOctF32><<<grid, 128, smem, s>>>(fps, tvp, slots, Astr, Kstr, slot_elems, smem_k, buf); break;
        case kBrickOctF32: tv_sweep_kernel<kBrickOctF32><<<grid, 128, smem, s>>>(fps, tvp, slots, Astr, Kstr, slot_elems, smem_k, buf); break;
        case kTex3dF32: tv_sweep_kernel<kTex3dF32><<<grid, 128, smem, s>>>(fps, tvp, slots, Astr, Kstr, slot_elems, smem_k, buf); break;
        case kMortonOctF32: tv_sweep_kernel<kMortonOctF32><<<grid, 128, smem, s>>>(fps, tvp, slots, Astr, Kstr, slot_elems, smem_k, buf); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace nsl
