// runtime.cu — NEXT-2/3: six-way relighting, composite and depth-based
// obstacle shadow (R1-R3): the paper's shading pass after the
// network (PAPER.md L213-225 directional interpolation and composite; L458-462
// smoke-shell depth vs the obstacle's shadow map).  One thread per pixel,
// grid-stride, HBM-streaming: two float4 of maps + the depth in, one float4 out
// (the shadow-map texels are few and L2-resident).
#include <cuda_fp16.h>

#include "nsl_internal.cuh"

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
__device__ __forceinline__ void axes(const nsl_camera& c, double f[3], double r[3], double u[3]) {
    double F[3] = {c.forward[0], c.forward[1], c.forward[2]}, U[3] = {c.up[0], c.up[1], c.up[2]};
    const double nf = __dsqrt_rn(dot3(F, F));
    for (int a = 0; a < 3; ++a) f[a] = dd(F[a], nf);
    double x[3];
    cross3(f, U, x);
    const double nx = __dsqrt_rn(dot3(x, x));
    for (int a = 0; a < 3; ++a) r[a] = dd(x[a], nx);
    cross3(r, f, u);
}

// R1-R3 per-frame constants (fp64 -> fp32 once).  The unshadowed lights and the composite
// fold into one 3x8 matrix M over the pixel's eight channels; each shadowed light keeps its
// own weights and the affine map pixel -> (shadow pixel fi, fj, light depth z).
// One warp per frame, lane l < n_lights handles light l (the fp64 chains run in parallel);
// lane 0 sums M over the lights in light order.
constexpr int kSetupWarps = 4;
__global__ void __launch_bounds__(32 * kSetupWarps) relight_setup_kernel(const RelightIn* __restrict__ in, int F,
                                                                         int n_lights, RelightConst rc,
                                                                         RelightFrame* __restrict__ out) {
    const int fi = blockIdx.x * kSetupWarps + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (fi >= F) return;
    const RelightIn& ri = in[fi];
    const nsl_camera cam = ri.cam;
    RelightFrame& p = out[fi];
    double f[3], r[3], u[3];
    axes(cam, f, r, u);
    const double W = cam.width, H = cam.height;
    const double ay = dm((double)cam.extent, 0.5), ax = dd(dm(ay, W), H);
    const double cx = ds(dd(1.0, W), 1.0), cy = ds(1.0, dd(1.0, H)), ex = dd(2.0, W), ey = dd(-2.0, H);
    double W0[3], Ex[3], Ey[3];
    for (int a = 0; a < 3; ++a) {
        const double P = cam.position[a];
        W0[a] = da(da(P, dm(dm(cx, ax), r[a])), dm(dm(cy, ay), u[a]));
        Ex[a] = dm(dm(ex, ax), r[a]);
        Ey[a] = dm(dm(ey, ay), u[a]);
        if (lane == 0) {
            p.W0[a] = (float)(cam.projection == 0 ? W0[a] : P);
            p.F0[a] = (float)da(da(f[a], dm(dm(cx, ax), r[a])), dm(dm(cy, ay), u[a]));
            p.Ex[a] = (float)Ex[a];
            p.Ey[a] = (float)Ey[a];
        }
    }
    const int l = lane;
    const bool on = l < n_lights;
    const bool shadowed = on && ri.shadow_map[l] != nullptr;
    double w[8] = {};
    if (on) {
        double n[3] = {ri.lights[l].to_light[0], ri.lights[l].to_light[1], ri.lights[l].to_light[2]};
        const double nn = __dsqrt_rn(dot3(n, n));
        for (int a = 0; a < 3; ++a) n[a] = dd(n[a], nn);
        const float c[3] = {(float)dot3(n, r), (float)dot3(n, u), (float)(-dot3(n, f))};   // R1, rounded once
        w[c[0] > 0.0f ? 0 : 4] = c[0] > 0.0f ? c[0] : -c[0];
        w[c[1] > 0.0f ? 1 : 5] = c[1] > 0.0f ? c[1] : -c[1];
        w[c[2] > 0.0f ? 6 : 2] = c[2] > 0.0f ? c[2] : -c[2];
    }
    const unsigned smask = __ballot_sync(0xffffffffu, shadowed);
    if (shadowed) {
        RelightShadowed& S = p.sl[__popc(smask & ((1u << l) - 1u))];
        for (int ch = 0; ch < 8; ++ch) S.w[ch] = (float)w[ch];
        for (int k = 0; k < 3; ++k) S.rgb[k] = ri.lights[l].rgb[k];
        const nsl_camera sc = ri.shadow_cam[l];
        double sf[3], sr[3], su[3];
        axes(sc, sf, sr, su);
        const double say = dm((double)sc.extent, 0.5), sax = dd(dm(say, (double)sc.width), (double)sc.height);
        const double hw = dm(0.5, (double)sc.width), hh = dm(0.5, (double)sc.height);
        // fi = (a + 1) Ws/2 with a = (p - Ps).r_s / a_x;  fj = (1 - b) Hs/2;  z = (p - Ps).f_s
        double G[3][3];                                  // gradient of (fi, fj, z) w.r.t. p
        for (int a = 0; a < 3; ++a) {
            G[0][a] = dm(dd(sr[a], sax), hw);
            G[1][a] = -dm(dd(su[a], say), hh);
            G[2][a] = sf[a];
        }
        const double off[3] = {hw, hh, 0.0};
        double O[3];                                     // ortho: W0; persp: camera position
        for (int a = 0; a < 3; ++a) O[a] = ds(cam.projection == 0 ? W0[a] : (double)cam.position[a], sc.position[a]);
        for (int o = 0; o < 3; ++o) {
            S.q[o][0] = (float)da(off[o], dot3(O, G[o]));
            S.q[o][1] = (float)dot3(Ex, G[o]);
            S.q[o][2] = (float)dot3(Ey, G[o]);
            S.q[o][3] = (float)dot3(f, G[o]);
            for (int a = 0; a < 3; ++a) S.g[o][a] = (float)G[o][a];
        }
        S.Ws = sc.width;
        S.Hs = sc.height;
        S.map = ri.shadow_map[l];
    }
    // M = composite + sum over unshadowed lights, in light order (lane 0)
    double rgb[3] = {0.0, 0.0, 0.0};
    if (on && !shadowed)
        for (int k = 0; k < 3; ++k) rgb[k] = ri.lights[l].rgb[k];
    double M[3][8];
    for (int k = 0; k < 3; ++k)
        for (int ch = 0; ch < 8; ++ch) M[k][ch] = ch == 3 ? (double)rc.bg[k] : ch == 7 ? (double)rc.emis[k] : 0.0;
    for (int j = 0; j < 4; ++j) {
        double wj[8], rj[3];
        for (int ch = 0; ch < 8; ++ch) wj[ch] = __shfl_sync(0xffffffffu, w[ch], j);
        for (int k = 0; k < 3; ++k) rj[k] = __shfl_sync(0xffffffffu, rgb[k], j);
        for (int k = 0; k < 3; ++k)
            for (int ch = 0; ch < 8; ++ch) M[k][ch] = da(M[k][ch], dm(rj[k], wj[ch]));
    }
    if (lane == 0) {
        for (int k = 0; k < 3; ++k)
            for (int ch = 0; ch < 8; ++ch) p.M[k][ch] = (float)M[k][ch];
        p.ns = __popc(smask);
        p.projection = cam.projection;
    }
}

constexpr int kRelightThreads = 256;
#ifndef NSL_RL_SH_PPT           // relight with shadow maps: pixels per thread, CTAs per SM
#define NSL_RL_SH_PPT 1
#endif
#ifndef NSL_RL_SH_MINB
#define NSL_RL_SH_MINB 8
#endif

// One CTA = kRelightThreads*PPT consecutive pixels of one frame; the frame's constants are
// staged to shared memory once.  Maps/depth are streamed (evict-first), the output is written
// with streaming stores; only the shadow maps stay in cache.  Two configurations (measured,
// DESIGN.md §11): without shadow maps 4 pixels per thread (all loads issued together: 0.94 of
// the HBM copy peak); with shadow maps the depth -> shadow-texel chain is two dependent
// round trips, so 1 pixel per thread at full occupancy hides it better (+9 %).
template <int PPT, int MINB>
__global__ void __launch_bounds__(kRelightThreads, MINB) relight_kernel(const RelightFrame* __restrict__ frames,
                                                                  RelightConst rc, int blocks_per_frame,
                                                                  const float4* __restrict__ maps,
                                                                  const float* __restrict__ depth,
                                                                  float4* __restrict__ out) {
    __shared__ RelightFrame fs;
    const int f = blockIdx.x / blocks_per_frame;
    const int chunk = blockIdx.x - f * blocks_per_frame;
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(frames + f);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&fs);
        for (int i = threadIdx.x; i < (int)(sizeof(RelightFrame) / 4); i += kRelightThreads) dst[i] = src[i];
    }
    __syncthreads();
    const int npf = rc.W * rc.H;
    const size_t fbase = (size_t)f * npf;
    const int p0 = chunk * (kRelightThreads * PPT) + threadIdx.x;
    float4 m0[PPT], m1[PPT];
    float D[PPT];
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int pix = p0 + k * kRelightThreads;
        if (pix < npf) {
            const size_t q = fbase + pix;
            m0[k] = __ldcs(maps + 2 * q);
            m1[k] = __ldcs(maps + 2 * q + 1);
            D[k] = depth ? __ldcs(depth + q) : 0.0f;
        }
    }
    const int ns = fs.ns;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int pix = p0 + k * kRelightThreads;
        if (pix >= npf) break;
        const float ch[8] = {m0[k].x, m0[k].y, m0[k].z, m0[k].w, m1[k].x, m1[k].y, m1[k].z, m1[k].w};
        float o[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float acc = 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j) acc = fmaf(fs.M[c][j], ch[j], acc);
            o[c] = acc;
        }
        if (ns > 0) {
            const float px = (float)(pix % rc.W), py = (float)(pix / rc.W);
            float dir[3] = {0.0f, 0.0f, 0.0f};
            if (fs.projection != 0 && D[k] > 0.0f) {
#pragma unroll
                for (int a = 0; a < 3; ++a) dir[a] = fmaf(py, fs.Ey[a], fmaf(px, fs.Ex[a], fs.F0[a]));
                const float inv = rsqrtf(fmaf(dir[0], dir[0], fmaf(dir[1], dir[1], dir[2] * dir[2])));
#pragma unroll
                for (int a = 0; a < 3; ++a) dir[a] *= inv;
            }
#pragma unroll
            for (int l = 0; l < 4; ++l) {       // ns <= 4: unrolled, so the shadow-map loads overlap
                if (l >= ns) break;
                const RelightShadowed& S = fs.sl[l];
                float s = 0.0f;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j != 3 && j != 7) s = fmaf(S.w[j], ch[j], s);
                float v = 1.0f;
                if (D[k] > 0.0f) {                                      // R3 depth shadow
                    float t[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float kd = fs.projection == 0
                                             ? S.q[c][3]
                                             : fmaf(dir[0], S.g[c][0], fmaf(dir[1], S.g[c][1], dir[2] * S.g[c][2]));
                        const float lin = fs.projection == 0 ? fmaf(py, S.q[c][2], fmaf(px, S.q[c][1], S.q[c][0]))
                                                             : S.q[c][0];
                        t[c] = fmaf(D[k], kd, lin);
                    }
                    if (t[0] >= 0.0f && t[1] >= 0.0f && t[0] < (float)S.Ws && t[1] < (float)S.Hs) {
                        const float zs = __ldg(S.map + (size_t)(int)t[1] * S.Ws + (int)t[0]);
                        if (zs + rc.bias < t[2]) v = 0.0f;
                    }
                }
                const float w = v * s;
#pragma unroll
                for (int c = 0; c < 3; ++c) o[c] = fmaf(S.rgb[c], w, o[c]);
            }
        }
        __stcs(out + fbase + pix, make_float4(o[0], o[1], o[2], 1.0f - m0[k].w));
    }
}

}  // namespace

cudaError_t launch_relight(const RelightIn* in, int F, int n_lights, RelightFrame* frames, const RelightConst& rc,
                           const float4* maps, const float* depth, float4* out, cudaStream_t s) {
    relight_setup_kernel<<<(F + kSetupWarps - 1) / kSetupWarps, 32 * kSetupWarps, 0, s>>>(in, F, n_lights, rc, frames);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const long long per = kRelightThreads * (rc.any_shadow ? NSL_RL_SH_PPT : 4);
    const long long bpf = ((long long)rc.W * rc.H + per - 1) / per;
    if (bpf * F >= (1LL << 31)) return cudaErrorInvalidConfiguration;
    if (rc.any_shadow)
        relight_kernel<NSL_RL_SH_PPT, NSL_RL_SH_MINB><<<(unsigned)(bpf * F), kRelightThreads, 0, s>>>(frames, rc, (int)bpf, maps, depth, out);
    else
        relight_kernel<4, 1><<<(unsigned)(bpf * F), kRelightThreads, 0, s>>>(frames, rc, (int)bpf, maps, depth, out);
    return cudaGetLastError();
}

// Compact host output (nsl_guiding_map_host_f16): the fp32 guiding map packed to fp16 (RNE) on
// the device before the PCIe download, 10 B per pixel instead of 20.  One thread per pixel,
// 16-B loads / 8-B stores, HBM-bound.
__global__ void __launch_bounds__(256) pack_half_kernel(const float4* __restrict__ rgbt, const float* __restrict__ depth,
                                                        uint2* __restrict__ rgbt_h, __half* __restrict__ depth_h,
                                                        size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 v = __ldcs(rgbt + i);
    const __half2 a = __floats2half2_rn(v.x, v.y), b = __floats2half2_rn(v.z, v.w);
    uint2 o;
    o.x = *reinterpret_cast<const uint32_t*>(&a);
    o.y = *reinterpret_cast<const uint32_t*>(&b);
    __stcs(rgbt_h + i, o);
    depth_h[i] = __float2half_rn(__ldcs(depth + i));
}

cudaError_t launch_pack_half(const float* rgbt, const float* depth, uint16_t* rgbt_h, uint16_t* depth_h, size_t n,
                             cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    pack_half_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(reinterpret_cast<const float4*>(rgbt), depth,
                                                                  reinterpret_cast<uint2*>(rgbt_h),
                                                                  reinterpret_cast<__half*>(depth_h), n);
    return cudaGetLastError();
}

}  // namespace nsl
