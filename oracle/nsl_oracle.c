/* oracle/nsl_oracle.c — plain, slow, single-threaded CPU oracle of the
 * guiding-map ray march.  TEST INFRASTRUCTURE ONLY (see nsl_oracle.h).
 *
 * Written step by step from DESIGN.md §2 (canonical C1-C14), which restates
 * PAPER.md Algorithm 1 (L394-407), eq:approx (L361-365) and §4.2 (L410).
 * Build with -ffp-contract=off so that every fp32 expression below is
 * evaluated exactly as written (fmaf() is the C99 correctly-rounded fma).
 */
#include "nsl_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <stddef.h>
#include <string.h>

#ifndef M_PI /* strict ISO C modes do not define it (same value as glibc's) */
#define M_PI 3.14159265358979323846
#endif

/* ---------------------------------------------------------------- C10 HG */
/* Henyey-Greenstein phase ("Henyey-Greenstein phase function
 * with g=0"; formula SPEC S:59): (1-g^2) / (4 pi (1+g^2-2 g c)^(3/2)). */
double orc_hg(double g, double c) {
    double d = (1.0 + g * g) - 2.0 * g * c;
    return (1.0 - g * g) / ((4.0 * M_PI) * (d * sqrt(d)));
}

/* ---------------------------------------------------------------- C4 jitter */
/* MurmurHash3 finaliser. */
uint32_t orc_fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

/* Alg. 1 line "x0 <- x0 + delta; delta: random jitter",
 * keyed per (seed, frame, pixel) — DESIGN.md C4. */
uint32_t orc_jitter_hash(uint64_t seed, uint32_t frame_id, uint32_t pixel) {
    uint32_t lo = (uint32_t)(seed & 0xffffffffu), hi = (uint32_t)(seed >> 32);
    uint32_t h = orc_fmix32(lo ^ 0x9E3779B9u);
    h = orc_fmix32(h ^ hi);
    h = orc_fmix32(h ^ frame_id);
    h = orc_fmix32(h ^ pixel);
    return h;
}

float orc_jitter_delta(const orc_march* m, uint32_t frame_id, uint32_t pixel) {
    if (!m->jitter) return 0.0f;
    uint32_t h = orc_jitter_hash(m->seed, frame_id, pixel);
    float u = (float)(h >> 8) * (1.0f / 16777216.0f);   /* exact: 24-bit integer times 2^-24 */
    return u * m->step;                                  /* one fp32 multiply */
}

/* ---------------------------------------------------------------- C1 sampler */
/* Voxel (i,j,k) (0-based) of the x-fastest grid; padded index 0 and n+1 are
 * the zero apron ("outside the grid is vacuum", DESIGN.md ledger #15). */
static double padded_voxel(const orc_grid* g, const float* vals, int i, int j, int k) {
    if (i < 1 || j < 1 || k < 1 || i > g->nx || j > g->ny || k > g->nz) return 0.0;
    size_t idx = ((size_t)(k - 1) * (size_t)g->ny + (size_t)(j - 1)) * (size_t)g->nx + (size_t)(i - 1);
    return (double)vals[idx];
}

static int inside_support(const orc_grid* g, const float u[3]) {
    return u[0] > 0.0f && u[0] < (float)(g->nx + 1) &&
           u[1] > 0.0f && u[1] < (float)(g->ny + 1) &&
           u[2] > 0.0f && u[2] < (float)(g->nz + 1);
}

static double lerp64(double a, double b, double t) { return a + t * (b - a); }

/* Trilinear reconstruction of sigma_s's carrier "in a 3D texture"
 * (PAPER.md L410), border-zero, interpolating x, then y, then z (C1). */
double orc_sample(const orc_grid* g, const float* vals, const float u[3]) {
    if (!inside_support(g, u)) return 0.0;
    float fl0 = floorf(u[0]), fl1 = floorf(u[1]), fl2 = floorf(u[2]);
    int i = (int)fl0, j = (int)fl1, k = (int)fl2;
    double fx = (double)(u[0] - fl0), fy = (double)(u[1] - fl1), fz = (double)(u[2] - fl2);
    double c000 = padded_voxel(g, vals, i, j, k), c100 = padded_voxel(g, vals, i + 1, j, k);
    double c010 = padded_voxel(g, vals, i, j + 1, k), c110 = padded_voxel(g, vals, i + 1, j + 1, k);
    double c001 = padded_voxel(g, vals, i, j, k + 1), c101 = padded_voxel(g, vals, i + 1, j, k + 1);
    double c011 = padded_voxel(g, vals, i, j + 1, k + 1), c111 = padded_voxel(g, vals, i + 1, j + 1, k + 1);
    double x00 = lerp64(c000, c100, fx), x10 = lerp64(c010, c110, fx);
    double x01 = lerp64(c001, c101, fx), x11 = lerp64(c011, c111, fx);
    double y0 = lerp64(x00, x10, fy), y1 = lerp64(x01, x11, fy);
    return lerp64(y0, y1, fz);
}

/* ---------------------------------------------------------------- C3 frame constants */
static double dot3(const double a[3], const double b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
static void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
static double norm3(const double a[3]) { return sqrt(dot3(a, a)); }

int orc_frame_constants_compute(const orc_grid* g, const orc_camera* cam,
                                const orc_light* lights, int32_t n_lights, int32_t light_mode,
                                const orc_medium* med, const orc_march* m,
                                orc_frame_constants* out) {
    (void)m;
    if (!g || !cam || !med || !out || n_lights < 1 || n_lights > 4) return 1;
    memset(out, 0, sizeof(*out));
    double dx = (double)g->voxel_width;
    double F[3] = {cam->forward[0], cam->forward[1], cam->forward[2]};
    double Up[3] = {cam->up[0], cam->up[1], cam->up[2]};
    double nf = norm3(F);
    double f[3] = {F[0] / nf, F[1] / nf, F[2] / nf};
    double c[3];
    cross3(f, Up, c);
    double nc = norm3(c);
    double r[3] = {c[0] / nc, c[1] / nc, c[2] / nc};
    double u[3];
    cross3(r, f, u);
    double W = (double)cam->width, H = (double)cam->height;
    double ay = (double)cam->extent * 0.5;
    double ax = (ay * W) / H;
    double cx = 1.0 / W - 1.0, cy = 1.0 - 1.0 / H;
    double ex = 2.0 / W, ey = -2.0 / H;
    out->inv_dx = (float)(1.0 / dx);
    for (int a = 0; a < 3; ++a) {
        double P = (double)cam->position[a], o = (double)g->origin[a];
        /* ortho: origin(px,py) = P + s_x ax r + s_y ay u, to padded index space */
        double w = P + (cx * ax) * r[a];
        w = w + (cy * ay) * u[a];
        out->B[a] = (float)((w - o) / dx + 0.5);
        out->Dg[a] = (float)(f[a] / dx);
        /* persp */
        out->Oe[a] = (float)((P - o) / dx + 0.5);
        out->F0[a] = (float)((f[a] + (cx * ax) * r[a]) + (cy * ay) * u[a]);
        out->fwd[a] = (float)f[a];
        if (cam->projection == 0) {
            out->Ex[a] = (float)(((ex * ax) * r[a]) / dx);
            out->Ey[a] = (float)(((ey * ay) * u[a]) / dx);
        } else {
            out->Ex[a] = (float)((ex * ax) * r[a]);
            out->Ey[a] = (float)((ey * ay) * u[a]);
        }
    }
    /* lights: explicit list, or the surrogate set of eq:approx:
     * front = omega = -f, top = omega x z, bottom = -omega x z (normalised; #8) */
    double Ln[4][3];
    if (light_mode == 1) {
        if (n_lights > 3) return 1;
        double om[3] = {-f[0], -f[1], -f[2]};
        double A[3] = {m ? m->guide_axis[0] : 0.0, m ? m->guide_axis[1] : 0.0, m ? m->guide_axis[2] : 0.0};
        if (A[0] == 0.0 && A[1] == 0.0 && A[2] == 0.0) { A[2] = 1.0; }
        double nA = norm3(A);
        double a[3] = {A[0] / nA, A[1] / nA, A[2] / nA};
        double s[3];
        cross3(om, a, s);
        double ns = norm3(s);
        if (ns < 1e-6) {
            double xh[3] = {1.0, 0.0, 0.0};
            cross3(om, xh, s);
            ns = norm3(s);
        }
        double t[3] = {s[0] / ns, s[1] / ns, s[2] / ns};
        for (int q = 0; q < 3; ++q) {
            Ln[0][q] = om[q];
            Ln[1][q] = t[q];
            Ln[2][q] = -t[q];
        }
    } else {
        if (!lights) return 1;
        for (int l = 0; l < n_lights; ++l) {
            double L[3] = {lights[l].to_light[0], lights[l].to_light[1], lights[l].to_light[2]};
            double nl = norm3(L);
            for (int q = 0; q < 3; ++q) Ln[l][q] = L[q] / nl;
        }
    }
    for (int l = 0; l < n_lights; ++l) {
        for (int q = 0; q < 3; ++q) {
            out->Ln[l][q] = (float)Ln[l][q];
            out->Lg[l][q] = (float)(Ln[l][q] / dx);
        }
        /* phase angle between incoming propagation (-to_light) and outgoing (-dir): cos = to_light . dir */
        double P = orc_hg((double)med->hg_g, dot3(Ln[l], f));
        out->P64[l] = P;
        out->P[l] = (float)P;
    }
    return 0;
}

/* ---------------------------------------------------------------- C5-C12 march */
typedef struct {
    const orc_grid* g;
    const float* vals;
    orc_density_fn fn;
    void* ctx;
} dens_t;

static double density(const dens_t* d, const float u[3]) {
    if (!inside_support(d->g, u)) return 0.0;
    if (d->fn) return d->fn(u, d->ctx);
    return orc_sample(d->g, d->vals, u);
}

/* C8: light transmittance from U along light l, right-endpoint rule, no jitter,
 * to the support exit.  Returns T^l; *M gets the number of samples. */
static double light_march(const dens_t* d, const float U[3], const float Lg[3], float hl,
                          double kappa, uint32_t* M) {
    double sum_sigma_t = 0.0;
    uint32_t j = 1;
    for (;; ++j) {
        float s = (float)j * hl;
        float Y[3] = {fmaf(s, Lg[0], U[0]), fmaf(s, Lg[1], U[1]), fmaf(s, Lg[2], U[2])};
        if (!inside_support(d->g, Y)) break;
        sum_sigma_t += kappa * density(d, Y);
        if (j > 100000000u) break;   /* unreachable for |Lg| = 1/dx; guards a corrupt input */
    }
    *M = j - 1;
    return exp(-(double)hl * sum_sigma_t);
}

/* Conservative upper bound on the primary step index whose sample can lie in
 * the support box (fp64 slab test on a 1-voxel-expanded box). */
static int64_t primary_upper_bound(const orc_grid* g, const float O[3], const float D[3],
                                   float delta, float h) {
    double t0 = -1e300, t1 = 1e300;
    double n[3] = {g->nx, g->ny, g->nz};
    for (int a = 0; a < 3; ++a) {
        double lo = -1.0, hi = n[a] + 2.0;
        if (D[a] == 0.0f) {
            if (!((double)O[a] > lo && (double)O[a] < hi)) return 0;
            continue;
        }
        double ta = (lo - (double)O[a]) / (double)D[a], tb = (hi - (double)O[a]) / (double)D[a];
        if (ta > tb) { double tt = ta; ta = tb; tb = tt; }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
    }
    if (t1 < t0 || t1 <= 0.0) return 0;
    double nmax = floor((t1 - (double)delta) / (double)h) + 2.0;
    if (nmax < 0.0) return 0;
    if (nmax > 1e8) nmax = 1e8;
    return (int64_t)nmax;
}

/* ================================================================ NEXT-4: transmittance volume
 * DESIGN.md §12 (V2-V5), written out plainly in fp64: the lattice of the light
 * step vector, the line sums toward and away from the light, and the trilinear
 * lookup.  Test infrastructure only, like everything in this file. */
int orc_tv_lattice_compute(const orc_grid* g, const float Lg[3], float hl, orc_tv_lattice* L) {
    if (!g || !Lg || !L || !(hl > 0.0f)) return 1;
    for (int a = 0; a < 3; ++a) L->d[a] = (double)hl * (double)Lg[a];
    L->ell = norm3(L->d);
    if (!(L->ell > 0.0)) return 1;
    for (int a = 0; a < 3; ++a) L->dhat[a] = L->d[a] / L->ell;
    const double zh[3] = {0.0, 0.0, 1.0}, xh[3] = {1.0, 0.0, 0.0};
    double c[3];
    cross3(L->dhat, zh, c);
    if (norm3(c) < 1e-6) cross3(L->dhat, xh, c);
    const double nc = norm3(c);
    for (int a = 0; a < 3; ++a) L->e1[a] = c[a] / nc;
    cross3(L->dhat, L->e1, L->e2);
    const double n[3] = {g->nx + 1.0, g->ny + 1.0, g->nz + 1.0};
    double amin = 1e300, amax = -1e300, bmin = 1e300, bmax = -1e300, kmin = 1e300, kmax = -1e300;
    for (int corner = 0; corner < 8; ++corner) {
        const double p[3] = {(corner & 1) ? n[0] : 0.0, (corner & 2) ? n[1] : 0.0, (corner & 4) ? n[2] : 0.0};
        const double a = dot3(p, L->e1), b = dot3(p, L->e2), k = dot3(p, L->dhat) / L->ell;
        if (a < amin) amin = a;
        if (a > amax) amax = a;
        if (b < bmin) bmin = b;
        if (b > bmax) bmax = b;
        if (k < kmin) kmin = k;
        if (k > kmax) kmax = k;
    }
    L->a0 = (int64_t)floor(amin) - 1;
    L->A = (int64_t)ceil(amax) - L->a0 + 2;
    L->b0 = (int64_t)floor(bmin) - 1;
    L->B = (int64_t)ceil(bmax) - L->b0 + 2;
    L->k0 = (int64_t)floor(kmin) - 1;
    L->K = (int64_t)ceil(kmax) - L->k0 + 2;
    return 0;
}

int64_t orc_tv_index(const orc_tv_lattice* L, int64_t i, int64_t j, int64_t k) { return (j * L->K + k) * L->A + i; }

int orc_tv_build(const orc_grid* g, const float* vals, orc_density_fn density_fn, void* density_ctx,
                 const orc_tv_lattice* L, float hl, double kappa, double* tau_plus, double* tau_minus) {
    if (!g || (!vals && !density_fn) || !L || !tau_plus || !tau_minus) return 1;
    const dens_t dens = {g, vals, density_fn, density_ctx};
    double* rho = (double*)malloc(sizeof(double) * (size_t)L->K);
    if (!rho) return 1;
    for (int64_t j = 0; j < L->B; ++j)
        for (int64_t i = 0; i < L->A; ++i) {
            for (int64_t k = 0; k < L->K; ++k) {          /* V3 */
                float P[3];
                for (int a = 0; a < 3; ++a)
                    P[a] = (float)((double)(L->a0 + i) * L->e1[a] + (double)(L->b0 + j) * L->e2[a] +
                                   (double)(L->k0 + k) * L->d[a]);
                rho[k] = density(&dens, P);
            }
            double acc = 0.0;                              /* V4: tau- (k' < k) */
            for (int64_t k = 0; k < L->K; ++k) {
                tau_minus[orc_tv_index(L, i, j, k)] = kappa * (double)hl * acc;
                acc += rho[k];
            }
            acc = 0.0;                                     /* V4: tau+ (k' > k) */
            for (int64_t k = L->K - 1; k >= 0; --k) {
                tau_plus[orc_tv_index(L, i, j, k)] = kappa * (double)hl * acc;
                acc += rho[k];
            }
        }
    free(rho);
    return 0;
}

double orc_tv_lookup(const orc_tv_lattice* L, const double* tau, const float U[3]) {
    const double u[3] = {U[0], U[1], U[2]};
    const double f[3] = {dot3(u, L->e1) - (double)L->a0, dot3(u, L->e2) - (double)L->b0,
                         dot3(u, L->dhat) / L->ell - (double)L->k0};
    const int64_t lim[3] = {L->A - 2, L->B - 2, L->K - 2};
    int64_t c[3];
    double w[3];
    for (int a = 0; a < 3; ++a) {
        double fl = floor(f[a]);
        if (fl < 0.0) fl = 0.0;
        if (fl > (double)lim[a]) fl = (double)lim[a];
        c[a] = (int64_t)fl;
        w[a] = f[a] - fl;
    }
    double v = 0.0;
    for (int corner = 0; corner < 8; ++corner) {
        const int di = corner & 1, dj = (corner >> 1) & 1, dk = (corner >> 2) & 1;
        const double wt = (di ? w[0] : 1.0 - w[0]) * (dj ? w[1] : 1.0 - w[1]) * (dk ? w[2] : 1.0 - w[2]);
        v += wt * tau[orc_tv_index(L, c[0] + di, c[1] + dj, c[2] + dk)];
    }
    return v;
}

double orc_light_tau(const orc_grid* g, const float* vals, orc_density_fn density_fn, void* density_ctx,
                     const float U[3], const float Lg[3], float hl, double kappa) {
    const dens_t dens = {g, vals, density_fn, density_ctx};
    uint32_t M = 0;
    return -log(light_march(&dens, U, Lg, hl, kappa, &M));
}

/* C8's sample count M from U (no sampling): the leading in-support light samples. */
static uint32_t light_count(const orc_grid* g, const float U[3], const float Lg[3], float hl) {
    uint32_t j = 1;
    for (;; ++j) {
        float s = (float)j * hl;
        float Y[3] = {fmaf(s, Lg[0], U[0]), fmaf(s, Lg[1], U[1]), fmaf(s, Lg[2], U[2])};
        if (!inside_support(g, Y) || j > 100000000u) break;
    }
    return j - 1;
}

int orc_guiding_map(const orc_grid* g, const float* vals,
                    orc_density_fn density_fn, void* density_ctx,
                    const orc_camera* cam, const orc_light* lights, int32_t n_lights,
                    int32_t light_mode, const orc_medium* med, const orc_march* m,
                    uint32_t frame_id, int64_t n_pix, const int64_t* pix,
                    double* out_rgbt, float* out_depth, uint32_t* out_debug, double* out_margin,
                    const int32_t* forced_hit, const int32_t* forced_term, int32_t no_clip_n) {
    if (!g || (!vals && !density_fn) || !cam || !lights || !med || !m || !out_rgbt || !out_depth) return 1;
    if (g->nx < 1 || g->ny < 1 || g->nz < 1 || !(g->voxel_width > 0.0f)) return 1;
    if (cam->width < 1 || cam->height < 1 || !(m->step > 0.0f)) return 1;
    orc_frame_constants fc;
    if (orc_frame_constants_compute(g, cam, lights, n_lights, light_mode, med, m, &fc)) return 1;
    const int W = cam->width, H = cam->height;
    if (!pix) n_pix = (int64_t)W * H;
    const float h = m->step;
    const float hl = m->light_step > 0.0f ? m->light_step : m->step;
    const double kappa = (double)med->extinction, alpha = (double)med->albedo;
    const double g_hg = (double)med->hg_g;
    const dens_t dens = {g, vals, density_fn, density_ctx};
    /* NEXT-4 (DESIGN.md §12 V1): every light but the guide set's front light uses its own
     * transmittance volume; each is built here independently (the mirror lattice of an
     * opposite light included). */
    orc_tv_lattice tv_lat[4];
    double* tv_tau[4] = {NULL, NULL, NULL, NULL};
    double* tv_scratch = NULL;
    int tv_on[4] = {0, 0, 0, 0};
    if (m->light_model == 1) {
        for (int l = 0; l < n_lights; ++l) {
            if (light_mode == 1 && l == 0) continue;
            if (orc_tv_lattice_compute(g, fc.Lg[l], hl, &tv_lat[l])) return 1;
            const size_t cnt = (size_t)(tv_lat[l].A * tv_lat[l].B * tv_lat[l].K);
            tv_tau[l] = (double*)malloc(sizeof(double) * cnt);
            tv_scratch = (double*)realloc(tv_scratch, sizeof(double) * cnt);
            if (!tv_tau[l] || !tv_scratch) return 1;
            orc_tv_build(g, vals, density_fn, density_ctx, &tv_lat[l], hl, kappa, tv_tau[l], tv_scratch);
            tv_on[l] = 1;
        }
        free(tv_scratch);
    }

    for (int64_t q = 0; q < n_pix; ++q) {
        int64_t p = pix ? pix[q] : q;
        int px = (int)(p % W), py = (int)(p / W);
        /* C3: per-pixel ray in padded index space */
        float O[3], D[3], dir[3];
        if (cam->projection == 0) {
            for (int a = 0; a < 3; ++a) {
                O[a] = fmaf((float)py, fc.Ey[a], fmaf((float)px, fc.Ex[a], fc.B[a]));
                D[a] = fc.Dg[a];
                dir[a] = fc.fwd[a];
            }
        } else {
            float d[3];
            for (int a = 0; a < 3; ++a) d[a] = fmaf((float)py, fc.Ey[a], fmaf((float)px, fc.Ex[a], fc.F0[a]));
            float qn = fmaf(d[2], d[2], fmaf(d[1], d[1], d[0] * d[0]));
            float inv = 1.0f / sqrtf(qn);
            for (int a = 0; a < 3; ++a) {
                dir[a] = d[a] * inv;
                D[a] = dir[a] * fc.inv_dx;
                O[a] = fc.Oe[a];
            }
        }
        double P[4];
        for (int l = 0; l < n_lights; ++l) {
            if (cam->projection == 0) P[l] = fc.P64[l];
            else P[l] = orc_hg(g_hg, ((double)fc.Ln[l][0] * dir[0] + (double)fc.Ln[l][1] * dir[1]) +
                                         (double)fc.Ln[l][2] * dir[2]);
        }
        /* C4 */
        const float delta = orc_jitter_delta(m, frame_id, (uint32_t)((uint32_t)py * (uint32_t)W + (uint32_t)px));

        /* C5: n = 1 .. n_max, every n tested (the clip only bounds the loop) */
        int64_t n_max = no_clip_n > 0 ? (int64_t)no_clip_n : primary_upper_bound(g, O, D, delta, h);
        if (m->max_steps > 0 && n_max > m->max_steps) n_max = m->max_steps;
        int32_t f_hit = forced_hit ? forced_hit[q] : -1;
        int32_t f_term = forced_term ? forced_term[q] : -1;

        uint32_t n_lo = 0, n_hi = 0, n_hit = 0, n_term = 0, n_occ = 0, lsamp = 0;
        double S[4] = {0, 0, 0, 0};
        double tau = 0.0, T = 1.0;
        float Dout = 0.0f;
        double hit_margin = INFINITY, term_margin = INFINITY;
        int terminated = 0;
        for (int64_t n = 1; n <= n_max; ++n) {
            float t = fmaf((float)n, h, delta);
            float U[3] = {fmaf(t, D[0], O[0]), fmaf(t, D[1], O[1]), fmaf(t, D[2], O[2])};
            if (!inside_support(g, U)) continue;
            if (!n_lo) n_lo = (uint32_t)n;
            n_hi = (uint32_t)n;
            if (terminated) continue;              /* keep scanning only for n_hi (debug) */
            n_term = (uint32_t)n;
            double rho = density(&dens, U);
            if (rho > 0.0) {
                ++n_occ;
                double sigma_t = kappa * rho, sigma_s = alpha * sigma_t;
                /* C6 depth: first n with sigma_s > tau (Alg. 1 "if D = 0 and sigma_n > tau") */
                if (f_hit < 0) {
                    if (!n_hit) {
                        double mg = m->depth_tau > 0.0f ? fabs(sigma_s - (double)m->depth_tau) / (double)m->depth_tau
                                                        : fabs(sigma_s);
                        if (mg < hit_margin) hit_margin = mg;
                        if ((float)sigma_s > m->depth_tau) { n_hit = (uint32_t)n; Dout = t; }
                    }
                } else if ((int64_t)f_hit == n) {
                    n_hit = (uint32_t)n; Dout = t;
                }
                /* C7 transmittance and opacity */
                double s = sigma_t * (double)h;
                double T_prev = T;
                tau += s;
                T = exp(-tau);
                double A;
                if (m->opacity_form == 0) A = alpha * T_prev * (1.0 - exp(-s));
                else if (m->opacity_form == 1) A = alpha * T_prev * s;
                else A = T_prev * sigma_s;
                /* C8 + C10: L_n = sum_l T^l P_l (rgb applied at the end), L += A_n L_n */
                for (int l = 0; l < n_lights; ++l) {
                    uint32_t M = 0;
                    double Tl;
                    if (tv_on[l]) {                      /* NEXT-4 V5 lookup; V6: M still counted */
                        Tl = exp(-orc_tv_lookup(&tv_lat[l], tv_tau[l], U));
                        M = light_count(g, U, fc.Lg[l], hl);
                    } else {
                        Tl = light_march(&dens, U, fc.Lg[l], hl, kappa, &M);
                    }
                    lsamp += M;
                    S[l] += A * Tl;
                }
                /* C11 early termination */
                if (m->t_min > 0.0f) {
                    double mg = fabs(T - (double)m->t_min) / (double)m->t_min;
                    if (mg < term_margin) term_margin = mg;
                }
                if (f_term < 0) {
                    if ((float)T < m->t_min) terminated = 1;
                }
            }
            if (f_term >= 0 && (int64_t)f_term == n) terminated = 1;
        }
        double L[3] = {0, 0, 0};
        for (int c = 0; c < 3; ++c)
            for (int l = 0; l < n_lights; ++l) L[c] += (double)lights[l].rgb[c] * P[l] * S[l];
        out_rgbt[4 * q + 0] = L[0];
        out_rgbt[4 * q + 1] = L[1];
        out_rgbt[4 * q + 2] = L[2];
        out_rgbt[4 * q + 3] = T;
        out_depth[q] = Dout;
        if (out_debug) {
            uint32_t* o = out_debug + 6 * q;
            o[0] = n_lo; o[1] = n_hi; o[2] = n_hit; o[3] = n_term; o[4] = n_occ; o[5] = lsamp;
        }
        if (out_margin) {
            out_margin[2 * q + 0] = hit_margin;
            out_margin[2 * q + 1] = term_margin;
        }
    }
    for (int l = 0; l < 4; ++l) free(tv_tau[l]);
    return 0;
}

/* ================================================================ NEXT-1: six-way bake
 * DESIGN.md §10 (B1-B6): deterministic single-scatter estimator of the six-way
 * lightmaps ("{L_x^+, L_x^-, L_y^+, L_y^-, L_z^+, L_z^-}", L477
 * "single bounce ... g = 0 ... samples per pixel"), transparency (L255) and an
 * emissive carrier; jittered fixed-step quadrature with counter-based RNG. */

static void camera_axes(const orc_camera* cam, double f[3], double r[3], double u[3]) {
    double F[3] = {cam->forward[0], cam->forward[1], cam->forward[2]};
    double Up[3] = {cam->up[0], cam->up[1], cam->up[2]};
    double nf = norm3(F);
    for (int a = 0; a < 3; ++a) f[a] = F[a] / nf;
    double c[3];
    cross3(f, Up, c);
    double nc = norm3(c);
    for (int a = 0; a < 3; ++a) r[a] = c[a] / nc;
    cross3(r, f, u);
}

/* B2: counter-based stream keyed by (seed, frame, pixel, sample) */
void orc_bake_random(uint64_t seed, uint32_t frame, uint32_t pixel, uint32_t sample, float u_out[4]) {
    uint32_t h = orc_fmix32((uint32_t)(seed & 0xffffffffu) ^ 0x85EBCA6Bu);
    h = orc_fmix32(h ^ (uint32_t)(seed >> 32));
    h = orc_fmix32(h ^ frame);
    h = orc_fmix32(h ^ pixel);
    h = orc_fmix32(h ^ sample);
    for (int i = 0; i < 4; ++i) {
        u_out[i] = (float)(h >> 8) * (1.0f / 16777216.0f);
        h = orc_fmix32(h + 0x9E3779B9u);
    }
}

/* B1: billboard-axis light directions n_l (fp64) in the packing order of B6:
 * right +r, top +u, back f, left -r, bottom -u, front -f. */
static void bake_lights(const orc_camera* cam, double n[6][3]) {
    double f[3], r[3], u[3];
    camera_axes(cam, f, r, u);
    for (int a = 0; a < 3; ++a) {
        n[0][a] = r[a];
        n[1][a] = u[a];
        n[2][a] = f[a];
        n[3][a] = -r[a];
        n[4][a] = -u[a];
        n[5][a] = -f[a];
    }
}

int orc_bake_light_constants(const orc_grid* g, const orc_camera* cam, float Lg[6][3], float Ln[6][3]) {
    if (!g || !cam) return 1;
    double n[6][3];
    bake_lights(cam, n);
    for (int l = 0; l < 6; ++l)
        for (int a = 0; a < 3; ++a) {
            Ln[l][a] = (float)n[l][a];
            Lg[l][a] = (float)(n[l][a] / (double)g->voxel_width);
        }
    return 0;
}

int orc_sixway_bake(const orc_grid* g, const float* vals, orc_density_fn density_fn, void* density_ctx,
                    const orc_camera* cam, const orc_medium* med, const orc_bake* b, uint32_t frame_id,
                    int64_t n_pix, const int64_t* pix, double* out8, uint32_t* out_steps) {
    if (!g || (!vals && !density_fn) || !cam || !med || !b || !out8) return 1;
    if (b->spp < 1 || !(b->step > 0.0f) || !(b->light_step > 0.0f)) return 1;
    const orc_light dummy[1] = {{{1.0f, 0.0f, 0.0f}, {1.0f, 1.0f, 1.0f}}};
    orc_march m0;
    memset(&m0, 0, sizeof m0);
    m0.step = b->step;
    orc_frame_constants fc;
    if (orc_frame_constants_compute(g, cam, dummy, 1, 0, med, &m0, &fc)) return 1;
    double n6[6][3];
    bake_lights(cam, n6);
    float Lg[6][3], Ln[6][3];
    orc_bake_light_constants(g, cam, Lg, Ln);
    const int W = cam->width, H = cam->height;
    if (!pix) n_pix = (int64_t)W * H;
    const float hb = b->step, hbl = b->light_step;
    const double kappa = (double)med->extinction, alpha = (double)med->albedo, ghg = (double)med->hg_g;
    const dens_t dens = {g, vals, density_fn, density_ctx};

    for (int64_t q = 0; q < n_pix; ++q) {
        int64_t p = pix ? pix[q] : q;
        int px = (int)(p % W), py = (int)(p / W);
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t steps = 0;
        for (int s = 0; s < b->spp; ++s) {
            float u4[4];
            orc_bake_random(b->seed, frame_id, (uint32_t)p, (uint32_t)s, u4);
            const float fx = (float)px + (u4[0] - 0.5f), fy = (float)py + (u4[1] - 0.5f);
            float O[3], D[3], dir[3];
            if (cam->projection == 0) {
                for (int a = 0; a < 3; ++a) {
                    O[a] = fmaf(fy, fc.Ey[a], fmaf(fx, fc.Ex[a], fc.B[a]));
                    D[a] = fc.Dg[a];
                    dir[a] = fc.fwd[a];
                }
            } else {
                float d[3];
                for (int a = 0; a < 3; ++a) d[a] = fmaf(fy, fc.Ey[a], fmaf(fx, fc.Ex[a], fc.F0[a]));
                float qn = fmaf(d[2], d[2], fmaf(d[1], d[1], d[0] * d[0]));
                float inv = 1.0f / sqrtf(qn);
                for (int a = 0; a < 3; ++a) {
                    dir[a] = d[a] * inv;
                    D[a] = dir[a] * fc.inv_dx;
                    O[a] = fc.Oe[a];
                }
            }
            double P[6];
            for (int l = 0; l < 6; ++l)
                P[l] = orc_hg(ghg, ((double)Ln[l][0] * dir[0] + (double)Ln[l][1] * dir[1]) + (double)Ln[l][2] * dir[2]);
            const float o2 = u4[2] * hb, o3 = u4[3] * hbl;
            /* k = 0 .. k_max; every k tested (the bound only limits the loop) */
            int64_t k_max = primary_upper_bound(g, O, D, o2, hb) + 1;
            if (b->max_steps > 0 && k_max > b->max_steps) k_max = b->max_steps;
            double tau = 0.0, sc[6] = {0, 0, 0, 0, 0, 0}, em = 0.0;
            for (int64_t k = 0; k <= k_max; ++k) {
                float t = fmaf((float)k, hb, o2);
                float U[3] = {fmaf(t, D[0], O[0]), fmaf(t, D[1], O[1]), fmaf(t, D[2], O[2])};
                if (!inside_support(g, U)) continue;
                ++steps;
                double rho = density(&dens, U);
                if (!(rho > 0.0)) continue;
                double sigma_t = kappa * rho;
                double Tk = exp(-tau);
                double wsc = alpha * sigma_t * (double)hb * Tk;          /* sigma_s h T_k */
                em += (1.0 - alpha) * sigma_t * (double)hb * Tk;           /* sigma_a h T_k */
                for (int l = 0; l < 6; ++l) {
                    double sum = 0.0;
                    for (uint32_t j = 1;; ++j) {
                        float sj = fmaf((float)(j - 1), hbl, o3);
                        float Y[3] = {fmaf(sj, Lg[l][0], U[0]), fmaf(sj, Lg[l][1], U[1]), fmaf(sj, Lg[l][2], U[2])};
                        if (!inside_support(g, Y)) break;
                        sum += kappa * density(&dens, Y);
                        if (j > 100000000u) break;
                    }
                    sc[l] += wsc * exp(-(double)hbl * sum) * P[l];
                }
                tau += sigma_t * (double)hb;
                if (b->t_min > 0.0f && (float)exp(-tau) < b->t_min) break;
            }
            /* B6 packing: (right, top, back, T) (left, bottom, front, E) */
            acc[0] += sc[0];
            acc[1] += sc[1];
            acc[2] += sc[2];
            acc[3] += exp(-tau);
            acc[4] += sc[3];
            acc[5] += sc[4];
            acc[6] += sc[5];
            acc[7] += em;
        }
        for (int c = 0; c < 8; ++c) out8[8 * q + c] = acc[c] / (double)b->spp;
        if (out_steps) out_steps[q] = steps;
    }
    return 0;
}

/* ================================================================ NEXT-2/3: relight, composite, shadow
 * DESIGN.md §11 (R1-R3): directionally weighted interpolation of the six-way
 * maps, composite (L213-218), depth-based obstacle shadow
 * (L458-462).  fp64 arithmetic; the shadow test reports its decision margins. */

static void pixel_ray_world(const orc_camera* cam, double px, double py, double o[3], double dir[3]) {
    double f[3], r[3], u[3];
    camera_axes(cam, f, r, u);
    const double W = cam->width, H = cam->height;
    const double sx = 2.0 * (px + 0.5) / W - 1.0, sy = 1.0 - 2.0 * (py + 0.5) / H;
    const double ay = 0.5 * cam->extent, ax = ay * W / H;
    if (cam->projection == 0) {
        for (int a = 0; a < 3; ++a) {
            o[a] = cam->position[a] + sx * ax * r[a] + sy * ay * u[a];
            dir[a] = f[a];
        }
    } else {
        double d[3];
        for (int a = 0; a < 3; ++a) {
            o[a] = cam->position[a];
            d[a] = f[a] + sx * ax * r[a] + sy * ay * u[a];
        }
        double nd = norm3(d);
        for (int a = 0; a < 3; ++a) dir[a] = d[a] / nd;
    }
}

/* R1 per-light billboard components c = (n.r, n.u, -n.f), rounded to fp32 */
int orc_relight_weights(const orc_camera* cam, const orc_light* lights, int32_t n_lights, float c_out[][3]) {
    if (!cam || !lights || n_lights < 1) return 1;
    double f[3], r[3], u[3];
    camera_axes(cam, f, r, u);
    for (int l = 0; l < n_lights; ++l) {
        double n[3] = {lights[l].to_light[0], lights[l].to_light[1], lights[l].to_light[2]};
        double nn = norm3(n);
        for (int a = 0; a < 3; ++a) n[a] /= nn;
        c_out[l][0] = (float)dot3(n, r);
        c_out[l][1] = (float)dot3(n, u);
        c_out[l][2] = (float)(-dot3(n, f));
    }
    return 0;
}

int orc_relight(const orc_camera* cam, const float* maps8, const float* depth, const orc_light* lights,
                int32_t n_lights, const float bg[3], const float emis[3], const orc_camera* shadow_cams,
                const float* const* shadow_maps, float bias, int64_t n_pix, const int64_t* pix, double* out4,
                double* out_margin) {
    if (!cam || !maps8 || !lights || n_lights < 1 || n_lights > 4 || !bg || !emis || !out4) return 1;
    float c[4][3];
    orc_relight_weights(cam, lights, n_lights, c);
    const int W = cam->width, H = cam->height;
    if (!pix) n_pix = (int64_t)W * H;
    for (int64_t q = 0; q < n_pix; ++q) {
        const int64_t p = pix ? pix[q] : q;
        const float* m = maps8 + 8 * p;
        /* Fig. 2 packing: m0 right(+x) m1 top(+y) m2 back(-z) m3 T | m4 left(-x) m5 bottom(-y) m6 front(+z) m7 E */
        const double Lpos[3] = {m[0], m[1], m[6]}, Lneg[3] = {m[4], m[5], m[2]};
        const double T = m[3], E = m[7];
        double out[3] = {0, 0, 0};
        double margin = INFINITY;
        for (int l = 0; l < n_lights; ++l) {
            double S = 0.0;
            for (int a = 0; a < 3; ++a) {
                if (c[l][a] > 0.0f) S += (double)c[l][a] * Lpos[a];
                else if (c[l][a] < 0.0f) S += (double)(-c[l][a]) * Lneg[a];
            }
            double v = 1.0;
            if (shadow_cams && shadow_maps && shadow_maps[l] && depth && depth[p] > 0.0f) {
                const orc_camera* sc = &shadow_cams[l];
                double o[3], dir[3], pt[3];
                pixel_ray_world(cam, (double)(p % W), (double)(p / W), o, dir);
                for (int a = 0; a < 3; ++a) pt[a] = o[a] + (double)depth[p] * dir[a];
                double sf[3], sr[3], su[3];
                camera_axes(sc, sf, sr, su);
                double d[3] = {pt[0] - sc->position[0], pt[1] - sc->position[1], pt[2] - sc->position[2]};
                const double say = 0.5 * sc->extent, sax = say * sc->width / sc->height;
                const double a_ = dot3(d, sr) / sax, b_ = dot3(d, su) / say, z = dot3(d, sf);
                const double fi = (a_ + 1.0) * sc->width / 2.0, fj = (1.0 - b_) * sc->height / 2.0;
                const double i = floor(fi), j = floor(fj);
                double mg = fmin(fmin(fi - i, 1.0 - (fi - i)), fmin(fj - j, 1.0 - (fj - j)));
                if (i >= 0 && j >= 0 && i < sc->width && j < sc->height) {
                    const double zs = (double)shadow_maps[l][(size_t)j * sc->width + (size_t)i];
                    if (isfinite(zs)) {
                        mg = fmin(mg, fabs(zs + (double)bias - z) / fmax(fabs(z), 1.0));
                        if (zs + (double)bias < z) v = 0.0;
                    }
                }
                if (mg < margin) margin = mg;
            }
            for (int k = 0; k < 3; ++k) out[k] += (double)lights[l].rgb[k] * v * S;
        }
        for (int k = 0; k < 3; ++k) out4[4 * q + k] = out[k] + (double)emis[k] * E + T * (double)bg[k];
        out4[4 * q + 3] = 1.0 - T;
        if (out_margin) out_margin[q] = margin;
    }
    return 0;
}
