// march.cu — rows a2, a4-a8: the guiding-map ray march (Algorithm 1,
// L394-407; C3-C12) for sm_100a.
//
// One thread per pixel; a warp marches a coherent 8x4 pixel tile, a CTA a
// 16x8 tile (4 warps).  Grid (frame, tile column, tile row): frames fastest,
// whole tile rows together, rows and columns centre-out (or tiles first when
// the frames view different volumes).  Sample positions use only explicitly rounded fp32
// operations (__fmaf_rn, __fmul_rn) so that every index decision is
// bit-identical to the oracle (C14); values are fp32 with FMA
// lerps.  The step range is clipped exactly (C5) and each light march's
// length is computed exactly (C8) so the inner loops carry no bounds tests.
//
// Before gathering, every sample tests the volume's occupancy bitmask (L1
// resident): a sample whose cell lies in an all-zero block is exactly 0 (C1),
// so skipping its load changes no bit of the result.  Whole tiles whose rays
// miss the occupied box are culled by tile_cull_kernel beforehand (exact:
// DESIGN.md §6), so their CTAs only write the empty map.  The kernel is
// issue-bound (profiles/).
#include "sampler.cuh"

namespace nsl {
namespace {

#ifndef NSL_PAIRNEG
#define NSL_PAIRNEG 1
#endif
#ifndef NSL_PACKG3
#define NSL_PACKG3 1
#endif
#ifndef NSL_STCS
#define NSL_STCS 1   // streaming (evict-first) map stores: C2 -1.2 %, C4 -0.5 % (profiles/r2_ab19)
#endif

// Tile culling (exact, orthographic views): every ray of a tile is parallel to D_g with
// its origin within the tile radius r of the centre ray; if the centre ray misses a box expanded by
// r, no sample of the tile lies in the box.  bit 0: misses the occupied box (FAST:
// every sample outside it is exactly 0); bit 1: misses the support box (DEBUG/COUNTED,
// which report n_lo/n_hi: C5).  One thread per (frame, tile).
// One thread per (frame, tile); grid (tile blocks, frame), so a CTA's tiles share one frame and its
// volume's slab boxes are staged once in shared memory.
constexpr int kCullThreads = 256, kCullSlabs = 128;
__global__ void __launch_bounds__(kCullThreads) tile_cull_kernel(const FrameParams* __restrict__ fps, int F,
                                                                 int tiles_x, int tiles, TileCull* __restrict__ cull,
                                                                 int early_trigger) {
    __shared__ int4 s_box[kCullSlabs];                  // (x0, y0, x1, y1) blocks of each z-slab
    // PDL: for small batches the march may launch at once (its launch latency hides under this
    // grid); for large ones the trigger is implicit at exit, so the march's CTAs -- which would
    // wait, resident, on this grid -- do not take the SMs this kernel's CTAs still need
    // (measured: C2 -0.9 % late vs early).  Small batches also skip the range (below): the cull
    // kernel is then on a critical path of a few tens of us (C1's single frame: +10 % with it).
    if (early_trigger) pdl_trigger();
    pdl_wait();                        // the FrameParams of frame_setup_kernel (after the volume build)
    const int f = blockIdx.y, t = blockIdx.x * kCullThreads + threadIdx.x;
    const FrameParams& sp = fps[f];
    const int nbz = sp.occ_nbz;
    const bool staged = nbz <= kCullSlabs;
    const int* sl = reinterpret_cast<const int*>(sp.occ) + sp.slab_off;
    if (staged) {
        for (int bz = threadIdx.x; bz < nbz; bz += kCullThreads) {
            const int2 mn = __ldg(reinterpret_cast<const int2*>(sl + 2 * bz));
            const int2 mx = __ldg(reinterpret_cast<const int2*>(sl + 2 * nbz + 2 * bz));
            s_box[bz] = make_int4(mn.x, mn.y, mx.x, mx.y);
        }
    }
    __syncthreads();
    if (t >= tiles) return;
    const int tx = t % tiles_x, ty = t / tiles_x;
    const float cx = (float)(tx * kTileW) + 0.5f * (kTileW - 1), cy = (float)(ty * kTileH) + 0.5f * (kTileH - 1);
    float c[3], D[3], iD[3];
    float rr = 0.0f;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        c[q] = fmaf(cy, sp.Ey[q], fmaf(cx, sp.Ex[q], sp.B[q]));
        D[q] = sp.Dg[q];
        iD[q] = sp.invD[q];
        // tile radius in index units: half extents of the tile (+1 pixel) along E_x, E_y, +1 for rounding
        const float e = (0.5f * kTileW + 1.0f) * fabsf(sp.Ex[q]) + (0.5f * kTileH + 1.0f) * fabsf(sp.Ey[q]);
        rr = fmaf(e, e, rr);
    }
    rr = sqrtf(rr) * 1.001f + 1.0f;
    uint32_t bits = 0;
    for (int box = 0; box < 2; ++box) {
        float t0 = -3.0e38f, t1 = 3.0e38f;
        bool miss = false;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const float lo = box == 0 ? sp.alo[q] : 0.0f, hi = box == 0 ? sp.ahi[q] : sp.supp[q];
            slab(c[q] - lo + rr, D[q], iD[q], hi - lo + 2.0f * rr, 0.0f, t0, t1, miss);
        }
        if (miss || !(t0 <= t1) || t1 < 0.0f) bits |= 1u << box;
    }
    // [t0, t1]: the union of the centre ray's hits on every z-slab's 2-D box of occupied blocks,
    // each grown by rr on all sides.  A tile ray is the centre ray shifted by <= rr across the view,
    // so a sample of it inside an occupied block (hence inside its slab's box) has its t inside
    // the grown box's hit of the centre ray: samples outside [t0, t1] are exactly 0 (C1).  Only
    // the slabs the bundle crosses inside the occupied box are visited (its z extent +- rr there).
    float lo = 3.0e38f, hi = -3.0e38f;
    if (early_trigger && !(bits & 1u)) {                 // small batch: no range (the whole box)
        lo = -3.0e38f;
        hi = 3.0e38f;
    } else if (!(bits & 1u)) {
        const float B = (float)(1 << sp.occ_shift);
        // the bundle's z range inside the occupied box -> the slabs to visit
        float ta = -3.0e38f, tb = 3.0e38f;
        bool m2 = false;
#pragma unroll
        for (int q = 0; q < 3; ++q)
            slab(c[q] - sp.alo[q] + rr, D[q], iD[q], sp.ahi[q] - sp.alo[q] + 2.0f * rr, 0.0f, ta, tb, m2);
        const float za = fmaf(ta, D[2], c[2]), zb = fmaf(tb, D[2], c[2]);
        const float zlo = (D[2] == 0.0f ? c[2] : fminf(za, zb)) - rr - 1.0f;
        const float zhi = (D[2] == 0.0f ? c[2] : fmaxf(za, zb)) + rr + 1.0f;
        const int bz0 = max(0, (int)floorf(zlo / B)), bz1 = min(nbz - 1, (int)floorf(zhi / B));
        // per-axis affine forms of the grown slab faces: t(face) = (face - c) / D
        float k0[3], k1[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            k1[q] = B * iD[q];
            k0[q] = (-rr - c[q]) * iD[q];
        }
        const float w[3] = {2.0f * rr * iD[0], 2.0f * rr * iD[1], 2.0f * rr * iD[2]};
        for (int bz = bz0; bz <= bz1; ++bz) {
            int4 b4;
            if (staged) {
                b4 = s_box[bz];
            } else {
                const int2 mn = __ldg(reinterpret_cast<const int2*>(sl + 2 * bz));
                const int2 mx = __ldg(reinterpret_cast<const int2*>(sl + 2 * nbz + 2 * bz));
                b4 = make_int4(mn.x, mn.y, mx.x, mx.y);
            }
            if (b4.z < 0) continue;                   // an empty slab
            const float blo[3] = {(float)b4.x, (float)b4.y, (float)bz};
            const float bhi[3] = {(float)(b4.z + 1), (float)(b4.w + 1), (float)(bz + 1)};
            float t0 = -3.0e38f, t1 = 3.0e38f;
            bool miss = false;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (D[q] != 0.0f) {
                    float u = fmaf(blo[q], k1[q], k0[q]), v = fmaf(bhi[q], k1[q], k0[q] + w[q]);
                    if (u > v) {
                        const float tt = u;
                        u = v;
                        v = tt;
                    }
                    t0 = fmaxf(t0, u);
                    t1 = fminf(t1, v);
                } else {
                    miss |= !(c[q] > blo[q] * B - rr && c[q] < bhi[q] * B + rr);
                }
            }
            if (!miss && t0 <= t1) {
                lo = fminf(lo, t0);
                hi = fmaxf(hi, t1);
            }
        }
        // the affine forms round differently from the slab test: widen by a relative 1e-5 of the
        // magnitudes plus one index unit of t (|D| = 1/dx: t of one index unit is dx) for safety
        const float pad = 1e-5f * fmaxf(fabsf(lo), fabsf(hi)) + 1.0f / sp.inv_dx;   // (no hit: stays empty)
        lo -= pad;
        hi += pad;
        if (!(lo <= hi)) bits |= 1u;       // no slab box on the bundle's path: FAST culls the tile too
    }
    TileCull out;
    out.t0 = lo;
    out.t1 = hi;
    out.bits = bits;
    out.pad = 0u;
    cull[(size_t)f * tiles + t] = out;
}

// NEXT-4 V5: trilinear lookup of (tau+, tau-) at index-space position (x, y, z) in the
// lattice of slot t (fractions from the clamped cell, as in the oracle).
__device__ __forceinline__ float2 tv_lookup(const TvParams& t, const float2* __restrict__ base, int Astr, int Kstr,
                                            float x, float y, float z) {
    const float al = fmaf(z, t.e1[2], fmaf(y, t.e1[1], x * t.e1[0])) - t.a0;
    const float be = fmaf(z, t.e2[2], fmaf(y, t.e2[1], x * t.e2[0])) - t.b0;
    const float ga = fmaf(z, t.dk[2], fmaf(y, t.dk[1], x * t.dk[0])) - t.k0;
    const float fi = fminf(fmaxf(floorf(al), 0.0f), (float)(t.A - 2));
    const float fj = fminf(fmaxf(floorf(be), 0.0f), (float)(t.B - 2));
    const float fk = fminf(fmaxf(floorf(ga), 0.0f), (float)(t.K - 2));
    const float wi = al - fi, wj = be - fj, wk = ga - fk;
    // V5 lookups at occupied samples stay inside the swept window
    NSL_ASSERT(fi >= (float)t.i_lo && fi + 1.0f <= (float)t.i_hi && fj >= (float)t.j_lo &&
               fj + 1.0f <= (float)t.j_hi && fk >= (float)t.k_lo && fk + 1.0f <= (float)t.k_hi);
    const float2* p = base + ((int64_t)fj * Kstr + (int64_t)fk) * Astr + (int64_t)fi;
    const int64_t sj = (int64_t)Kstr * Astr;
    const float2 c000 = __ldg(p), c100 = __ldg(p + 1), c010 = __ldg(p + Astr), c110 = __ldg(p + Astr + 1);
    const float2 c001 = __ldg(p + sj), c101 = __ldg(p + sj + 1), c011 = __ldg(p + sj + Astr),
                 c111 = __ldg(p + sj + Astr + 1);
    float2 r;
    r.x = lerpf(lerpf(lerpf(c000.x, c100.x, wi), lerpf(c010.x, c110.x, wi), wk),
                lerpf(lerpf(c001.x, c101.x, wi), lerpf(c011.x, c111.x, wi), wk), wj);
    r.y = lerpf(lerpf(lerpf(c000.y, c100.y, wi), lerpf(c010.y, c110.y, wi), wk),
                lerpf(lerpf(c001.y, c101.y, wi), lerpf(c011.y, c111.y, wi), wk), wj);
    return r;
}

// NL: the light set fixed at compile time, so the paths it cannot take are compiled out and
// the kernel carries less state: 3 = the guide set (front + the exactly opposite top/bottom
// pair, pair12 by construction), 1 = one light (march or C9), 0 = any set (runtime).
// k-th index of [0, n) in centre-out order (ties: the lower index first): n odd m, m-1, m+1,
// m-2, ...; n even m-1, m, m-2, m+1, ... with m = n / 2.  A bijection of [0, n).
__device__ __forceinline__ int centre_out(int k, int n) {
    const int m = n >> 1, h = k >> 1;
    if (n & 1) return (k & 1) ? m - 1 - h : m + h;
    return (k & 1) ? m + h : m - 1 - h;
}

template <int LAYOUT, int PROJ, int MODE, bool TV, int NL>
__global__ void __launch_bounds__(kThreads, (NL == 3 ? (TV ? NSL_MINB_G3TV : NSL_MINB_G3) : NL == 1 ? NSL_MINB_L1 : NSL_MINB) * 256 / kThreads) march_kernel(const FrameParams* __restrict__ fps, const MarchConst mc,
                                                         float4* __restrict__ out_rgbt, float* __restrict__ out_depth,
                                                         uint32_t* __restrict__ out_debug,
                                                         unsigned long long* __restrict__ counters, int W, int H,
                                                         const TileCull* __restrict__ cull, int tiles_x, TvArgs tv) {
    constexpr bool DEBUG = MODE == kDebug, COUNT = MODE == kCounted;
    // 3-D grid (frame, tile column rank, tile row rank): frames fastest, then the tiles of one
    // tile row, then rows -- rows and columns centre-out (centre_out), so whole tile rows run
    // together (the horizontal light lines of a row stay in one z-slab of the volume) and the
    // heavy centre tiles start first.  frame_major (frames of different volumes): (column, row,
    // frame), the CTAs in flight then cover one frame and share its volume.  No order table:
    // the tile follows from the block index without a dependent load.
    const bool fmaj = mc.frame_major != 0;
    const int f = (int)(fmaj ? blockIdx.z : blockIdx.x);
    const int tiles_y = (int)(fmaj ? gridDim.y : gridDim.z);
    const int tx = centre_out((int)(fmaj ? blockIdx.x : blockIdx.y), tiles_x);
    const int ty = centre_out((int)(fmaj ? blockIdx.y : blockIdx.z), tiles_y);
    pdl_wait();                        // launched with PDL after frame_setup / tile_cull: their outputs
    const FrameParams& sp = fps[f];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * kTileW + (warp % kWarpsX) * kWarpW + lane % kWarpW;
    const int py = ty * kTileH + (warp / kWarpsX) * kWarpH + lane / kWarpW;
    const bool valid = px < W && py < H;
    const size_t o = ((size_t)f * (size_t)H + (size_t)py) * (size_t)W + px;

    // the cull flag and the volume fields are independent loads: issue them together
    float tr0 = -3.0e38f, tr1 = 3.0e38f;               // the tile's occupied-slab range (FAST/COUNTED)
    uint32_t cflag = 0u;
    if (PROJ == 0) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(cull + (size_t)f * (tiles_x * tiles_y) + ty * tiles_x + tx));
        tr0 = q.x;
        tr1 = q.y;
        cflag = __float_as_uint(q.z);
    }
    Vol v;
    v.data = sp.data;
    v.sy = sp.sy;
    v.sz = sp.sz;
    v.occ = sp.occ;
    v.shift = sp.occ_shift;
    v.nbx = sp.occ_nbx;
    v.nby = sp.occ_nby;
    v.sx1 = sp.supp[0];
    v.sy1 = sp.supp[1];
    v.sz1 = sp.supp[2];
    v.mask_words = sp.slab_off;
    if (PROJ == 0 && (cflag & (DEBUG || COUNT ? 2 : 1))) {
        if (valid) {                   // the empty map: L = 0, T = 1, D = 0, counters 0
#if NSL_STCS
            __stcs(out_rgbt + o, make_float4(0.0f, 0.0f, 0.0f, 1.0f));
            __stcs(out_depth + o, 0.0f);
#else
            out_rgbt[o] = make_float4(0.0f, 0.0f, 0.0f, 1.0f);
            out_depth[o] = 0.0f;
#endif
            if (DEBUG) {
                uint32_t* dbg = out_debug + o * 6;
                dbg[0] = dbg[1] = dbg[2] = dbg[3] = dbg[4] = dbg[5] = 0u;
            }
        }
        return;                        // uniform over the CTA
    }
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
            for (int l = 0; l < 4; ++l) P[l] = 0.0f;     // ortho: per-frame phase, read at the end
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
        r.delta = mc.jitter ? jitter_delta(fmix32(sp.jh ^ pix), mc.h) : 0.0f;   // C4 (per-frame prefix sp.jh)

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
#if NSL_TILE_RANGE
            if (PROJ == 0 && !DEBUG) {               // the tile's occupied-slab range (tile_cull_kernel)
                u0 = fmaxf(u0, tr0);
                u1 = fminf(u1, tr1);
            }
#endif
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
        const bool paired = NL == 3 || (NL == 0 && sp.pair12 != 0);
        const int n_lights = NL ? NL : mc.n_lights;
        // positions from (float)n (one ALU I2FP per step): a separate float counter is spilled at 40
        // registers (a local load + load + store per primary step; C2 march -1.3 %)
        for (int n = m_lo; n <= m_hi; ++n) {
            float t, x, y, z;
            r.atf((float)n, t, x, y, z);
            if (COUNT) ++c_tp;
            const float rho = sample<LAYOUT, COUNT>(v, x, y, z, c_gath);
            if (rho > 0.0f) {
                ++n_occ;
                // C6/C7/C11 decide integers from sig_s and T: explicitly rounded ops, so every
                // kernel variant (FAST, DEBUG, COUNTED; any light set) takes the same decisions
                const float sig_t = __fmul_rn(mc.kappa, rho);
                const float sig_s = __fmul_rn(mc.alpha, sig_t);
                // C6 (t_n >= h > 0, so D == 0 <=> no hit yet: the FAST kernels keep no n_hit)
                if ((DEBUG ? n_hit == 0 : Dout == 0.0f) && sig_s > mc.tau_d) {
                    n_hit = n;
                    Dout = t;
                }
                const float s = __fmul_rn(sig_t, mc.h);  // C7
                const float Tp = T;
                tau = __fadd_rn(tau, s);
                T = __expf(-tau);
                float A;
                if (mc.form == NSL_OPACITY_EXP) A = mc.alpha * (Tp - T);
                else if (mc.form == NSL_OPACITY_RIEMANN) A = mc.alpha * Tp * s;
                else A = Tp * sig_s;
                const float kl = mc.hl * mc.kappa;
                const bool guide = mc.light_mode == NSL_LIGHTS_GUIDE;
                float2 tv0 = make_float2(0.0f, 0.0f);      // NEXT-4: the guide pair's (tau+, tau-)
                if (TV && guide && mc.n_lights > 1)
                    tv0 = tv_lookup(tv.params[f * tv.slots], tv.buf + (int64_t)f * tv.slots * tv.slot_elems,
                                    tv.Astr, tv.Kstr, x, y, z);
                if (!TV && paired) {                       // C8: top/bottom in one loop
                    int Ma, Mb, ma, mb;
                    float l1x = sp.Lg[1][0], l1y = sp.Lg[1][1], l1z = sp.Lg[1][2];   // (FAST: packed loads)
                    bool hzp = ((sp.lz0 >> 1) & 3) == 3;
                    if (DEBUG || COUNT) {
                        Ma = light_count(v, x, y, z, sp.Lg[1][0], sp.Lg[1][1], sp.Lg[1][2], mc.hl, sp.lim[1], sp.ilh[1]);
                        Mb = light_count(v, x, y, z, sp.Lg[2][0], sp.Lg[2][1], sp.Lg[2][2], mc.hl, sp.lim[2], sp.ilh[2]);
                        float ra[3], rb[3];
                        pair_regions(sp, v, z, ra, rb);
                        ma = min(Ma, box_count(x, y, z, ra, sp.ilh[1]));
                        mb = min(Mb, box_count(x, y, z, rb, sp.ilh[2]));
                    } else {
                        Ma = Mb = 0;
#if NSL_PAIRNEG && NSL_PACKG3
                        // the pair's constants by three vector loads (FrameParams.pk_*), light 2 = -light 1
                        // bit for bit (pair12), hence 1/(L2 h_l) = -1/(L1 h_l) exactly where L1 != 0
                        const int4 pg = sp.pk_geo;
                        const float4 pl = sp.pk_l1;
                        const float2 pi = *reinterpret_cast<const float2*>(&sp.pk_i1);
                        l1x = pl.x;
                        l1y = pl.y;
                        l1z = pl.z;
                        const float i1[3] = {pl.w, pi.x, pi.y};
                        const float i2[3] = {l1x != 0.0f ? -i1[0] : i1[0], l1y != 0.0f ? -i1[1] : i1[1],
                                             l1z != 0.0f ? -i1[2] : i1[2]};
                        float ra[3], rb[3];
                        pair_regions_pk(sp, v, z, pg, l1x, l1y, ra, rb);
                        ma = light_bound(v, x, y, z, l1x, l1y, l1z, mc.hl, i1, ra);
                        mb = light_bound(v, x, y, z, -l1x, -l1y, -l1z, mc.hl, i2, rb);
                        hzp = ((pg.z >> 1) & 3) == 3;
#elif NSL_PAIRNEG
                        float ra[3], rb[3];
                        pair_regions(sp, v, z, ra, rb);
                        const float i1[3] = {sp.ilh[1][0], sp.ilh[1][1], sp.ilh[1][2]};
                        const float i2[3] = {l1x != 0.0f ? -i1[0] : i1[0], l1y != 0.0f ? -i1[1] : i1[1],
                                             l1z != 0.0f ? -i1[2] : i1[2]};
                        ma = light_bound(v, x, y, z, l1x, l1y, l1z, mc.hl, i1, ra);
                        mb = light_bound(v, x, y, z, -l1x, -l1y, -l1z, mc.hl, i2, rb);
#else
                        float ra[3], rb[3];
                        pair_regions(sp, v, z, ra, rb);
                        ma = light_bound(v, x, y, z, sp.Lg[1][0], sp.Lg[1][1], sp.Lg[1][2], mc.hl, sp.ilh[1], ra);
                        mb = light_bound(v, x, y, z, sp.Lg[2][0], sp.Lg[2][1], sp.Lg[2][2], mc.hl, sp.ilh[2], rb);
#endif
                    }
                    if (COUNT) c_tl += (uint32_t)(ma + mb);
                    float sa, sb;
                    if (NSL_HZ && hzp)                         // both side lights horizontal: hoisted z plane
                        light_sum_pair_hz<LAYOUT, COUNT>(v, x, y, z, l1x, l1y, mc.hl, ma, mb, sa, sb, c_gath);
                    else
                        light_sum_pair<LAYOUT, COUNT>(v, x, y, z, l1x, l1y, l1z, mc.hl, ma, mb, sa, sb, c_gath);
                    S[1] = __fmaf_rn(A, __expf(-kl * sa), S[1]);
                    S[2] = __fmaf_rn(A, __expf(-kl * sb), S[2]);
                    lsamp += (uint32_t)(Ma + Mb);
                }
#pragma unroll
                for (int l = 0; l < 4; ++l) {             // C8 + C10
                    if (l < n_lights && !(!TV && paired && (l == 1 || l == 2))) {
                        float Tl;
                        const float lx = sp.Lg[l][0], ly = sp.Lg[l][1], lz = sp.Lg[l][2];
                        if (l == 0 && front_fast) {
                            Tl = Tp;                      // C9: T^front_n = T_{n-1}
                            if (COUNT) lsamp += (uint32_t)light_count(v, x, y, z, lx, ly, lz, mc.hl, sp.lim[l], sp.ilh[l]);
                        } else if (TV && !(guide && l == 0)) {   // NEXT-4 V5 (V6: M still counted)
                            const float tau = guide ? (l == 1 ? tv0.x : tv0.y)
                                                    : tv_lookup(tv.params[f * tv.slots + l],
                                                                tv.buf + ((int64_t)f * tv.slots + l) * tv.slot_elems,
                                                                tv.Astr, tv.Kstr, x, y, z).x;
                            Tl = __expf(-tau);
                            if (DEBUG || COUNT)
                                lsamp += (uint32_t)light_count(v, x, y, z, lx, ly, lz, mc.hl, sp.lim[l], sp.ilh[l]);
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
                                mm = light_bound(v, x, y, z, lx, ly, lz, mc.hl, sp.ilh[l], rl);
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
            if (l < n_lights) {
                const float w = (PROJ == 0 ? sp.P[l] : P[l]) * S[l];
                L0 += sp.rgb[l][0] * w;
                L1 += sp.rgb[l][1] * w;
                L2 += sp.rgb[l][2] * w;
            }
        }
        // the output offset again (cheaper than keeping it live through the march)
        const size_t oo = ((size_t)f * (size_t)H + (size_t)py) * (size_t)W + px;
#if NSL_STCS
        __stcs(out_rgbt + oo, make_float4(L0, L1, L2, T));   // streaming stores: the maps do not
        __stcs(out_depth + oo, Dout);                          // displace the volume in L2
#else
        out_rgbt[oo] = make_float4(L0, L1, L2, T);
        out_depth[oo] = Dout;
#endif
        const bool hit_support = n_lo > 0 && n_hi >= n_lo;
        if (DEBUG) {
            uint32_t* dbg = out_debug + oo * 6;
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

// Small batches (a single frame, the paper's per-frame use): one warp per 8x4 tile leaves
// most of the GPU idle and the time is the longest ray's serial light marches.  The split march
// gives each 8x4 tile kSplit warps: every warp runs the tile's primary march (cheap, identical),
// warp w takes the light marches of the occupied samples k with k % kSplit == w and parks their
// transmittances T^l_k in shared memory; warp 0 then folds S_l = fma(A_k, T^l_k, S_l) in k order
// -- the same operations in the same order as march_kernel's FAST guide-set path, so the maps are
// bitwise those of march_kernel (tests/test_gpu_parity.py test_split_march_is_bitwise_identical).
constexpr int kSplit = 4;
constexpr int kSplitMaxK = 96;                     // 4 x 96 x 32 floats = 48 KB of shared memory
template <int LAYOUT>
__global__ void __launch_bounds__(32 * kSplit) march_split_kernel(const FrameParams* __restrict__ fps,
                                                                  const MarchConst mc, float4* __restrict__ out_rgbt,
                                                                  float* __restrict__ out_depth, int W, int H,
                                                                  const TileCull* __restrict__ cull, int tiles_x,
                                                                  int tiles_y) {
    extern __shared__ float s_split[];            // [4][K][32]: A_k, T^0_k, T^1_k, T^2_k
    const int K = mc.split_k;
    const int f = (int)blockIdx.z;
    pdl_wait();                                    // FrameParams and the cull records
    const FrameParams& sp = fps[f];
    const int wv = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x0 = (int)blockIdx.x * kWarpW, y0 = (int)blockIdx.y * kWarpH;
    const int px = x0 + lane % kWarpW, py = y0 + lane / kWarpW;
    const int tx = x0 / kTileW, ty = y0 / kTileH;  // the 16x8 cull tile holding this 8x4 tile
    const bool valid = px < W && py < H;
    const float4 q = __ldg(reinterpret_cast<const float4*>(cull + (size_t)f * (tiles_x * tiles_y) + ty * tiles_x + tx));
    if (__float_as_uint(q.z) & 1u) {               // culled (uniform over the CTA): the empty map
        if (wv == 0 && valid) {
            const size_t o = ((size_t)f * (size_t)H + (size_t)py) * (size_t)W + px;
            out_rgbt[o] = make_float4(0.0f, 0.0f, 0.0f, 1.0f);
            out_depth[o] = 0.0f;
        }
        return;
    }
    Vol v;
    v.data = sp.data;
    v.sy = sp.sy;
    v.sz = sp.sz;
    v.occ = sp.occ;
    v.shift = sp.occ_shift;
    v.nbx = sp.occ_nbx;
    v.nby = sp.occ_nby;
    v.sx1 = sp.supp[0];
    v.sy1 = sp.supp[1];
    v.sz1 = sp.supp[2];
    v.mask_words = sp.slab_off;
    float* sA = s_split;
    float* sT = s_split + (size_t)K * 32;          // T^l_k at sT[(l * K + k) * 32 + lane]
    float T = 1.0f, Dout = 0.0f;
    int k = 0;
    uint32_t gdummy = 0;
    if (valid) {
        Ray r;
        const float fpx = (float)px, fpy = (float)py;
        r.ox = __fmaf_rn(fpy, sp.Ey[0], __fmaf_rn(fpx, sp.Ex[0], sp.B[0]));
        r.oy = __fmaf_rn(fpy, sp.Ey[1], __fmaf_rn(fpx, sp.Ex[1], sp.B[1]));
        r.oz = __fmaf_rn(fpy, sp.Ey[2], __fmaf_rn(fpx, sp.Ex[2], sp.B[2]));
        r.dx = sp.Dg[0];
        r.dy = sp.Dg[1];
        r.dz = sp.Dg[2];
        const float inv[3] = {sp.invD[0], sp.invD[1], sp.invD[2]};
        r.h = mc.h;
        const uint32_t pix = (uint32_t)py * (uint32_t)W + (uint32_t)px;
        r.delta = mc.jitter ? jitter_delta(fmix32(sp.jh ^ pix), mc.h) : 0.0f;   // C4
        // C5 as march_kernel's FAST path: the occupied box's step range (tile range applied), exact ends
        int m_lo = 1, m_hi = 0;
        {
            float u0 = -3.0e38f, u1 = 3.0e38f;
            bool miss = false;
            slab(r.ox - sp.alo[0], r.dx, inv[0], sp.ahi[0] - sp.alo[0], 1e-3f, u0, u1, miss);
            slab(r.oy - sp.alo[1], r.dy, inv[1], sp.ahi[1] - sp.alo[1], 1e-3f, u0, u1, miss);
            slab(r.oz - sp.alo[2], r.dz, inv[2], sp.ahi[2] - sp.alo[2], 1e-3f, u0, u1, miss);
#if NSL_TILE_RANGE
            u0 = fmaxf(u0, q.x);
            u1 = fminf(u1, q.y);
#endif
            if (!miss && u0 <= u1) {
                const float inv_h = 1.0f / mc.h;
                const float a = fmaxf(floorf((u0 - r.delta) * inv_h) - 1.0f, 1.0f);
                const float b = fminf(ceilf((u1 - r.delta) * inv_h) + 1.0f, (float)mc.Ncap);
                if (a <= b) {
                    m_lo = (int)a;
                    m_hi = (int)b;
                    while (m_lo <= m_hi && !r.in(v, m_lo)) ++m_lo;
                    while (m_hi >= m_lo && !r.in(v, m_hi)) --m_hi;
                }
            }
        }
        float tau = 0.0f;
        const bool front_fast = sp.front_ok && m_lo <= m_hi && !r.in(v, 1);   // C9 per ray
        const float kl = mc.hl * mc.kappa;
        for (int n = m_lo; n <= m_hi; ++n) {
            float t, x, y, z;
            r.atf((float)n, t, x, y, z);
            const float rho = sample<LAYOUT, false>(v, x, y, z, gdummy);
            if (rho > 0.0f) {
                const float sig_t = __fmul_rn(mc.kappa, rho);
                const float sig_s = __fmul_rn(mc.alpha, sig_t);
                if (Dout == 0.0f && sig_s > mc.tau_d) Dout = t;           // C6
                const float s = __fmul_rn(sig_t, mc.h);                  // C7
                const float Tp = T;
                tau = __fadd_rn(tau, s);
                T = __expf(-tau);
                float A;
                if (mc.form == NSL_OPACITY_EXP) A = mc.alpha * (Tp - T);
                else if (mc.form == NSL_OPACITY_RIEMANN) A = mc.alpha * Tp * s;
                else A = Tp * sig_s;
                NSL_ASSERT(k < K);
                if (wv == 0) sA[k * 32 + lane] = A;
                if (k % kSplit == wv) {                                  // this warp's light marches
                    float ra[3], rb[3];
                    pair_regions(sp, v, z, ra, rb);
                    const int ma = light_bound(v, x, y, z, sp.Lg[1][0], sp.Lg[1][1], sp.Lg[1][2], mc.hl, sp.ilh[1], ra);
                    const int mb = light_bound(v, x, y, z, sp.Lg[2][0], sp.Lg[2][1], sp.Lg[2][2], mc.hl, sp.ilh[2], rb);
                    float sa, sb;
                    if (NSL_HZ && ((sp.lz0 >> 1) & 3) == 3)
                        light_sum_pair_hz<LAYOUT, false>(v, x, y, z, sp.Lg[1][0], sp.Lg[1][1], mc.hl, ma, mb, sa, sb,
                                                         gdummy);
                    else
                        light_sum_pair<LAYOUT, false>(v, x, y, z, sp.Lg[1][0], sp.Lg[1][1], sp.Lg[1][2], mc.hl, ma, mb,
                                                      sa, sb, gdummy);
                    float T0;
                    if (front_fast) {
                        T0 = Tp;                                             // C9
                    } else {
                        float rl[3];
                        march_region(sp, v, 0, z, rl);
                        const int mm = light_bound(v, x, y, z, sp.Lg[0][0], sp.Lg[0][1], sp.Lg[0][2], mc.hl,
                                                   sp.ilh[0], rl);
                        T0 = __expf(-kl * light_sum<LAYOUT, false>(v, x, y, z, sp.Lg[0][0], sp.Lg[0][1], sp.Lg[0][2],
                                                                    mc.hl, mm, gdummy));
                    }
                    sT[(0 * K + k) * 32 + lane] = T0;
                    sT[(1 * K + k) * 32 + lane] = __expf(-kl * sa);
                    sT[(2 * K + k) * 32 + lane] = __expf(-kl * sb);
                }
                ++k;
                if (T < mc.t_min) break;                                 // C11
            }
        }
    }
    __syncthreads();
    if (wv != 0 || !valid) return;
    // a6: S_l in k order with march_kernel's operations (light order within a sample is immaterial:
    // the three sums are independent), then L_c = sum_l rgb_lc P_l S_l and the stores
    float S[3] = {0.0f, 0.0f, 0.0f};
    for (int j = 0; j < k; ++j) {
        const float A = sA[j * 32 + lane];
#pragma unroll
        for (int l = 0; l < 3; ++l) S[l] = __fmaf_rn(A, sT[(l * K + j) * 32 + lane], S[l]);
    }
    float L0 = 0.0f, L1 = 0.0f, L2 = 0.0f;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        const float w = sp.P[l] * S[l];
        L0 += sp.rgb[l][0] * w;
        L1 += sp.rgb[l][1] * w;
        L2 += sp.rgb[l][2] * w;
    }
    const size_t o = ((size_t)f * (size_t)H + (size_t)py) * (size_t)W + px;
    out_rgbt[o] = make_float4(L0, L1, L2, T);
    out_depth[o] = Dout;
}

__global__ void jitter_debug_kernel(MarchConst mc, uint32_t frame, int n, uint32_t* hash, float* delta) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    uint32_t h = jitter_hash(mc.seed_lo, mc.seed_hi, frame, (uint32_t)p);
    hash[p] = h;
    delta[p] = mc.jitter ? jitter_delta(h, mc.h) : 0.0f;
}

template <int LAYOUT, int PROJ, int MODE>
cudaError_t launch_lpm(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, float4* rgbt, float* depth,
                       uint32_t* debug, unsigned long long* counters, TileCull* cull,
                       const TvArgs* tv, cudaStream_t s) {
    const int tiles_x = (W + kTileW - 1) / kTileW, tiles_y = (H + kTileH - 1) / kTileH, tiles = tiles_x * tiles_y;
    if (tiles > 65535) return cudaErrorInvalidConfiguration;
    if (PROJ == 0) {
        if (F > 65535) return cudaErrorInvalidConfiguration;
        static const long long early_tiles = [] {
            const char* e = getenv("NSL_CULL_EARLY_TILES");
            return e ? atoll(e) : (long long)(8 * kCullThreads);
        }();
        const int early = (long long)F * tiles <= early_tiles;
        cudaError_t e = launch_pdl(tile_cull_kernel, dim3((unsigned)((tiles + kCullThreads - 1) / kCullThreads), (unsigned)F),
                                   dim3(kCullThreads), 0, s, fp, F, tiles_x, tiles, cull, early);
        if (e != cudaSuccess) return e;
    }
    const unsigned txn = (unsigned)tiles_x, tyn = (unsigned)tiles_y;
    const dim3 grid = mc.frame_major ? dim3(txn, tyn, (unsigned)F) : dim3((unsigned)F, txn, tyn);
    if (tv) {
        if constexpr (MODE == kFast) {
            if (NSL_TV_G3 && mc.light_mode == NSL_LIGHTS_GUIDE && mc.n_lights == 3)
                return launch_pdl(march_kernel<LAYOUT, PROJ, MODE, true, 3>, grid, dim3(kThreads), 0, s, fp, mc,
                                  rgbt, depth, debug, counters, W, H, (const TileCull*)cull, tiles_x, *tv);
            if (NSL_TV_NL && mc.n_lights == 1)
                return launch_pdl(march_kernel<LAYOUT, PROJ, MODE, true, 1>, grid, dim3(kThreads), 0, s, fp, mc,
                                  rgbt, depth, debug, counters, W, H, (const TileCull*)cull, tiles_x, *tv);
        }
        return launch_pdl(march_kernel<LAYOUT, PROJ, MODE, true, 0>, grid, dim3(kThreads), 0, s, fp, mc, rgbt,
                          depth, debug, counters, W, H, (const TileCull*)cull, tiles_x, *tv);
    }
    if constexpr (MODE == kFast) {
        if constexpr (PROJ == 0 && LAYOUT != kTex3dF32) {
            if (mc.split_k > 0 && mc.light_mode == NSL_LIGHTS_GUIDE && mc.n_lights == 3) {
                const unsigned sx = (unsigned)((W + kWarpW - 1) / kWarpW), sy = (unsigned)((H + kWarpH - 1) / kWarpH);
                return launch_pdl(march_split_kernel<LAYOUT>, dim3(sx, sy, (unsigned)F), dim3(32 * kSplit),
                                  (size_t)4 * mc.split_k * 32 * sizeof(float), s, fp, mc, rgbt, depth, W, H,
                                  (const TileCull*)cull, tiles_x, tiles_y);
            }
        }
        if (NSL_G3 && mc.light_mode == NSL_LIGHTS_GUIDE && mc.n_lights == 3)
            return launch_pdl(march_kernel<LAYOUT, PROJ, MODE, false, 3>, grid, dim3(kThreads), 0, s, fp, mc, rgbt,
                              depth, debug, counters, W, H, (const TileCull*)cull, tiles_x, TvArgs{});
        if (NSL_L1 && mc.n_lights == 1)
            return launch_pdl(march_kernel<LAYOUT, PROJ, MODE, false, 1>, grid, dim3(kThreads), 0, s, fp, mc, rgbt,
                              depth, debug, counters, W, H, (const TileCull*)cull, tiles_x, TvArgs{});
    }
    return launch_pdl(march_kernel<LAYOUT, PROJ, MODE, false, 0>, grid, dim3(kThreads), 0, s, fp, mc, rgbt, depth,
                      debug, counters, W, H, (const TileCull*)cull, tiles_x, TvArgs{});
}

template <int LAYOUT, int PROJ>
cudaError_t launch_lp(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, float4* rgbt, float* depth,
                      uint32_t* debug, unsigned long long* counters, TileCull* cull,
                      const TvArgs* tv, cudaStream_t s) {
    if (debug) return launch_lpm<LAYOUT, PROJ, kDebug>(fp, mc, F, W, H, rgbt, depth, debug, counters, cull, tv, s);
    if (counters)
        return launch_lpm<LAYOUT, PROJ, kCounted>(fp, mc, F, W, H, rgbt, depth, debug, counters, cull, tv, s);
    return launch_lpm<LAYOUT, PROJ, kFast>(fp, mc, F, W, H, rgbt, depth, debug, counters, cull, tv, s);
}

template <int LAYOUT>
cudaError_t launch_l(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, int proj, float4* rgbt,
                     float* depth, uint32_t* debug, unsigned long long* counters, TileCull* cull,
                     const TvArgs* tv, cudaStream_t s) {
    return proj == 0 ? launch_lp<LAYOUT, 0>(fp, mc, F, W, H, rgbt, depth, debug, counters, cull, tv, s)
                     : launch_lp<LAYOUT, 1>(fp, mc, F, W, H, rgbt, depth, debug, counters, cull, tv, s);
}

}  // namespace

int march_tile_w() { return kTileW; }
int march_split_max_k() { return kSplitMaxK; }
int march_tile_h() { return kTileH; }

size_t march_cull_bytes(int F, int W, int H) {
    return (size_t)F * ((W + kTileW - 1) / kTileW) * ((H + kTileH - 1) / kTileH) * sizeof(TileCull);
}

cudaError_t launch_march(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, int projection, int layout,
                         float4* rgbt, float* depth, uint32_t* debug, unsigned long long* counters,
                         TileCull* cull, const TvArgs* tv, cudaStream_t s) {
    switch (layout) {
        case kLinearF32: return launch_l<kLinearF32>(fp, mc, F, W, H, projection, rgbt, depth, debug, counters, cull, tv, s);
        case kQuadF32: return launch_l<kQuadF32>(fp, mc, F, W, H, projection, rgbt, depth, debug, counters, cull, tv, s);
        case kCornerF16: return launch_l<kCornerF16>(fp, mc, F, W, H, projection, rgbt, depth, debug, counters, cull, tv, s);
        case kOctF32: return launch_l<kOctF32>(fp, mc, F, W, H, projection, rgbt, depth, debug, counters, cull, tv, s);
        case kBrickOctF32: return launch_l<kBrickOctF32>(fp, mc, F, W, H, projection, rgbt, depth, debug, counters, cull, tv, s);
        case kTex3dF32: return launch_l<kTex3dF32>(fp, mc, F, W, H, projection, rgbt, depth, debug, counters, cull, tv, s);
        case kMortonOctF32: return launch_l<kMortonOctF32>(fp, mc, F, W, H, projection, rgbt, depth, debug, counters, cull, tv, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_jitter_debug(const MarchConst& mc, uint32_t frame_id, int n, uint32_t* hash, float* delta,
                                cudaStream_t s) {
    jitter_debug_kernel<<<(n + 255) / 256, 256, 0, s>>>(mc, frame_id, n, hash, delta);
    return cudaGetLastError();
}

}  // namespace nsl
