// setup.cu — rows a2/a3 per frame: camera frame constants, guide-light frame
// and phase (C3, C3b, C10), one thread per frame.
//
// Evaluated in fp64 with explicitly rounded operations (__dmul_rn, __dadd_rn,
// __dsub_rn, __ddiv_rn, __dsqrt_rn: no FMA contraction) in exactly the
// operation order DESIGN.md C3 prescribes, then rounded once to fp32, so that
// the per-pixel ray positions downstream are reproducible bit for bit.
#include "nsl_internal.cuh"

namespace nsl {
namespace {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }

// |a| = sqrt((ax ax + ay ay) + az az)
__device__ __forceinline__ double norm3(const double a[3]) {
    return __dsqrt_rn(da(da(dm(a[0], a[0]), dm(a[1], a[1])), dm(a[2], a[2])));
}
// (a x b)_x = ay bz - az by (cyclic)
__device__ __forceinline__ void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = ds(dm(a[1], b[2]), dm(a[2], b[1]));
    o[1] = ds(dm(a[2], b[0]), dm(a[0], b[2]));
    o[2] = ds(dm(a[0], b[1]), dm(a[1], b[0]));
}
__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
    return da(da(dm(a[0], b[0]), dm(a[1], b[1])), dm(a[2], b[2]));
}

// Henyey-Greenstein (C10): (1-g^2) / (4 pi d sqrt d),
// d = (1 + g^2) - 2 g c
__device__ __forceinline__ double hg64(double g, double c) {
    double d = ds(da(1.0, dm(g, g)), dm(dm(2.0, g), c));
    return dd(ds(1.0, dm(g, g)), dm(dm(4.0, 3.141592653589793), dm(d, __dsqrt_rn(d))));
}

// One warp per frame: every lane evaluates the camera basis (and the guide set's t), lane a < 3
// the per-axis constants of axis a, lane l < 4 the constants of light l, so the fp64 divide /
// sqrt chains run side by side instead of one after another; each lane writes its own fields
// with exactly the operations (and order) of C3/C3b/C10, so every value is unchanged.
constexpr int kSetupWarps = 4;
__global__ void __launch_bounds__(32 * kSetupWarps) frame_setup_kernel(const FrameIn* __restrict__ in,
                                                                      const nsl_light* __restrict__ lights, int F,
                                                                      MarchConst mc, FrameParams* __restrict__ out) {
    pdl_trigger();                     // the march (PDL) may launch now; it waits for this grid
    const int fi = blockIdx.x * kSetupWarps + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (fi >= F) {
        pdl_wait();
        return;
    }
    const FrameIn& fr = in[fi];
    const nsl_camera& cam = fr.cam;
    FrameParams& p = out[fi];
    const int nx = fr.vol.nx, ny = fr.vol.ny, nz = fr.vol.nz;
    const float supp[3] = {(float)(nx + 1), (float)(ny + 1), (float)(nz + 1)};
    if (lane == 0) {                   // ---- volume and scalar fields
        p.data = fr.vol.data;
        p.layout = fr.vol.layout;
        p.nx = nx;
        p.ny = ny;
        p.nz = nz;
        layout_strides(p.layout, nx, ny, p.sy, p.sz);
        for (int q = 0; q < 3; ++q) p.supp[q] = supp[q];
        p.projection = cam.projection;
        p.W = cam.width;
        p.H = cam.height;
        p.frame_id = fr.frame_id;
        p.occ = fr.vol.occ;
        p.occ_shift = fr.vol.og.shift;
        p.occ_nbx = fr.vol.og.nbx;
        p.occ_nby = fr.vol.og.nby;
        p.occ_words = fr.vol.og.words_total;   // mask + slab boxes
        p.slab_off = fr.vol.og.words;
        p.occ_nbz = fr.vol.og.nbz;
        p.pad2[0] = p.pad2[1] = 0;
        // C4: h32 = fmix32(jh ^ pixel) with jh = fmix32(fmix32(fmix32(lo32(seed) ^ 0x9E3779B9) ^
        // hi32(seed)) ^ frame_id): the first three rounds depend on the frame only
        auto fmix = [](uint32_t h) {
            h ^= h >> 16;
            h *= 0x85ebca6bu;
            h ^= h >> 13;
            h *= 0xc2b2ae35u;
            h ^= h >> 16;
            return h;
        };
        p.jh = fmix(fmix(fmix(mc.seed_lo ^ 0x9E3779B9u) ^ mc.seed_hi) ^ fr.frame_id);
    }

    // ---- camera basis (C3), every lane
    const double dx = (double)fr.vol.dx;
    double Fw[3] = {cam.forward[0], cam.forward[1], cam.forward[2]};
    double Up[3] = {cam.up[0], cam.up[1], cam.up[2]};
    double nf = norm3(Fw);
    double f[3] = {dd(Fw[0], nf), dd(Fw[1], nf), dd(Fw[2], nf)};
    double c[3];
    cross3(f, Up, c);
    double nc = norm3(c);
    double r[3] = {dd(c[0], nc), dd(c[1], nc), dd(c[2], nc)};
    double u[3];
    cross3(r, f, u);
    const double W = (double)cam.width, H = (double)cam.height;
    const double ay = dm((double)cam.extent, 0.5);
    const double ax = dd(dm(ay, W), H);
    const double cx = ds(dd(1.0, W), 1.0), cy = ds(1.0, dd(1.0, H));
    const double ex = dd(2.0, W), ey = dd(-2.0, H);
    if (lane == 0) p.inv_dx = (float)dd(1.0, dx);
    float Dg = 0.0f;
    if (lane < 3) {                    // ---- axis a = lane
        const int a = lane;
        const double P = (double)cam.position[a], o = (double)fr.vol.origin[a];
        double w = da(P, dm(dm(cx, ax), r[a]));
        w = da(w, dm(dm(cy, ay), u[a]));
        p.B[a] = (float)da(dd(ds(w, o), dx), 0.5);
        Dg = (float)dd(f[a], dx);
        p.Dg[a] = Dg;
        p.Oe[a] = (float)da(dd(ds(P, o), dx), 0.5);
        p.F0[a] = (float)da(da(f[a], dm(dm(cx, ax), r[a])), dm(dm(cy, ay), u[a]));
        p.fwd[a] = (float)f[a];
        if (cam.projection == 0) {
            p.Ex[a] = (float)dd(dm(dm(ex, ax), r[a]), dx);
            p.Ey[a] = (float)dd(dm(dm(ey, ay), u[a]), dx);
        } else {
            p.Ex[a] = (float)dm(dm(ex, ax), r[a]);
            p.Ey[a] = (float)dm(dm(ey, ay), u[a]);
        }
        // estimate helper (never decides an index on its own)
        p.invD[a] = Dg != 0.0f ? 1.0f / Dg : 0.0f;
    }

    // ---- light l = lane (C3b): explicit, or the surrogate set of eq:approx
    const int l = lane;
    const bool on = l < mc.n_lights;
    double Ln[3] = {0.0, 0.0, 0.0};
    const nsl_light* L = lights + (size_t)fi * mc.n_lights;
    if (l < 4 && on) {
        if (mc.light_mode == NSL_LIGHTS_GUIDE) {
            double om[3] = {-f[0], -f[1], -f[2]};
            if (l == 0) {
                for (int q = 0; q < 3; ++q) Ln[q] = om[q];
            } else {
                double A[3] = {mc.axis[0], mc.axis[1], mc.axis[2]};
                if (A[0] == 0.0 && A[1] == 0.0 && A[2] == 0.0) A[2] = 1.0;
                double nA = norm3(A);
                double an[3] = {dd(A[0], nA), dd(A[1], nA), dd(A[2], nA)};
                double sv[3];
                cross3(om, an, sv);
                double ns = norm3(sv);
                if (ns < 1e-6) {
                    const double xh[3] = {1.0, 0.0, 0.0};
                    cross3(om, xh, sv);
                    ns = norm3(sv);
                }
                for (int q = 0; q < 3; ++q) {
                    const double t = dd(sv[q], ns);
                    Ln[q] = l == 1 ? t : -t;
                }
            }
        } else {
            double v[3] = {L[l].to_light[0], L[l].to_light[1], L[l].to_light[2]};
            double nl = norm3(v);
            for (int q = 0; q < 3; ++q) Ln[q] = dd(v[q], nl);
        }
    }
    float Lg[3] = {0.0f, 0.0f, 0.0f};
    if (l < 4) {
        for (int q = 0; q < 3; ++q) {
            Lg[q] = on ? (float)dd(Ln[q], dx) : 0.0f;
            p.Ln[l][q] = on ? (float)Ln[q] : 0.0f;
            p.Lg[l][q] = Lg[q];
            p.rgb[l][q] = on ? L[l].rgb[q] : 0.0f;
        }
        // cos theta = to_light . dir (C10); per frame for ortho (dir = f)
        p.P[l] = on ? (float)hg64((double)mc.g, dot3(Ln, f)) : 0.0f;
        float ilh[3];
        for (int q = 0; q < 3; ++q) {  // estimate helpers
            p.lim[l][q] = Lg[q] > 0.0f ? supp[q] : (Lg[q] < 0.0f ? 0.0f : 3.0e38f);
            ilh[q] = Lg[q] != 0.0f ? 1.0f / (Lg[q] * mc.hl) : 1.0f;
            p.ilh[l][q] = ilh[q];
        }
        if (l == 1) {
            p.pk_l1 = make_float4(Lg[0], Lg[1], Lg[2], ilh[0]);
            p.pk_i1 = make_float4(ilh[1], ilh[2], 0.0f, 0.0f);
        }
    }
    // ---- cross-lane predicates: C9 (front light exactly -D_g), the opposite guide pair, L_z == 0
    float Dga[3], Lg1[3], Lg2[3], Lg0[3];
    for (int q = 0; q < 3; ++q) {
        Dga[q] = __shfl_sync(0xffffffffu, Dg, q);
        Lg0[q] = __shfl_sync(0xffffffffu, Lg[q], 0);
        Lg1[q] = __shfl_sync(0xffffffffu, Lg[q], 1);
        Lg2[q] = __shfl_sync(0xffffffffu, Lg[q], 2);
    }
    const unsigned lz = __ballot_sync(0xffffffffu, l < 4 && on && Lg[2] == 0.0f);
    if (lane == 0) {
        bool ok = mc.front_identity && mc.light_mode == NSL_LIGHTS_GUIDE && cam.projection == 0 && mc.hl == mc.h;
        for (int q = 0; q < 3; ++q) ok = ok && (Lg0[q] == -Dga[q]);
        p.front_ok = ok ? 1 : 0;
        bool pair = mc.light_mode == NSL_LIGHTS_GUIDE && mc.n_lights == 3;
        for (int q = 0; q < 3; ++q) pair = pair && (Lg2[q] == -Lg1[q]);
        p.pair12 = pair ? 1 : 0;
        p.lz0 = (int32_t)(lz & 0xfu);   // horizontal light: marches stay in one z slab
        p.pk_geo = make_int4(fr.vol.og.words, fr.vol.og.nbz, p.lz0, p.pair12);
        if (mc.n_lights < 2) {
            p.pk_l1 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            p.pk_i1 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
    }
    // ---- occupied box in padded-index positions: cells [bmin*B, (bmax+1)*B) -> U in [lo, hi),
    //      clipped to the support
    pdl_wait();                        // launched with PDL after the volume build: the AABB is its output
    float alo[3], ahi[3];
    if (fr.vol.aabb) {
        const int B = 1 << fr.vol.og.shift;
        for (int q = 0; q < 3; ++q) {
            const int bmin = fr.vol.aabb[q], bmax = fr.vol.aabb[3 + q];
            if (bmin > bmax) {                      // empty volume: a point box
                alo[q] = 0.0f;
                ahi[q] = 0.0f;
            } else {
                alo[q] = (float)(bmin * B);
                ahi[q] = fminf((float)((bmax + 1) * B), supp[q]);
            }
        }
    } else {
        for (int q = 0; q < 3; ++q) {
            alo[q] = 0.0f;
            ahi[q] = supp[q];
        }
    }
    if (lane < 3) {
        p.alo[lane] = alo[lane];
        p.ahi[lane] = ahi[lane];
    }
    if (l < 4)
        for (int q = 0; q < 3; ++q) p.alim[l][q] = Lg[q] > 0.0f ? ahi[q] : (Lg[q] < 0.0f ? alo[q] : 3.0e38f);
}

}  // namespace

cudaError_t launch_frame_setup(const FrameIn* in, const nsl_light* lights, int F, const MarchConst& mc,
                               FrameParams* out, cudaStream_t s) {
    const int blocks = (F + kSetupWarps - 1) / kSetupWarps;
    return launch_pdl(frame_setup_kernel, dim3(blocks), dim3(32 * kSetupWarps), 0, s, in, lights, F, mc, out);
}

}  // namespace nsl
