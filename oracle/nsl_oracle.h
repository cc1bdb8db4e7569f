/* oracle/nsl_oracle.h — CPU ORACLE for the guiding-map ray march.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2604_03748_b200, libnsl.so) never links, loads or
 * calls it, and this oracle shares no code, header, table or helper with it.
 *
 * What it computes: Algorithm 1 of PAPER.md ("Ray-marching for Guiding Map",
 * L394-407) with h = 10 dx (L410) and the surrogate light set of eq:approx
 * (L361-365), in the canonical reading written out in DESIGN.md §2 (C1-C14).
 * Everything that decides an index (frame constants, jitter, sample
 * positions, floors, inside tests) is fp32 with exactly the prescribed
 * operations (C14); everything after the positions (trilinear
 * weights, sigma, exp, sums) is fp64.  Threshold decisions (depth tau,
 * early termination T_min) compare the fp32-rounded fp64 value with the
 * fp32 threshold, i.e. in the kernel's precision (C14).
 *
 * Pins: see tests/test_oracle_*.py (closed forms P2-P4, invariants P5-P8,
 * brute force P10-P11, HG P12, sampler P13, hash P14).  No function here is
 * "parity unpinned" except the literal reproduction of the paper's own
 * implementation, for which the paper prints no values.
 */
#ifndef NSL_ORACLE_H
#define NSL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { int32_t nx, ny, nz; float origin[3]; float voxel_width; } orc_grid;
typedef struct {
    int32_t projection;               /* 0 orthographic, 1 perspective */
    float position[3], forward[3], up[3];
    float extent;                     /* ortho: image-plane height; persp: 2 tan(fov_y/2) */
    int32_t width, height;
} orc_camera;
typedef struct { float to_light[3]; float rgb[3]; } orc_light;
typedef struct { float extinction, albedo, hg_g; } orc_medium;
typedef struct {
    float step, light_step;           /* h, h_l (0 -> h) */
    int32_t max_steps;                /* N, 0 -> unbounded */
    float depth_tau, t_min;
    int32_t opacity_form;             /* 0 EXP, 1 RIEMANN, 2 LITERAL */
    int32_t jitter;                   /* 0 off, 1 per-ray hash */
    uint64_t seed;
    float guide_axis[3];              /* world axis "z" of eq:approx; (0,0,0) -> (0,0,1) */
    int32_t light_model;              /* 0 canonical march (C8), 1 transmittance volume */
} orc_march;

/* Frame constants of DESIGN.md C3 (fp64 evaluation, rounded once to fp32). */
typedef struct {
    float inv_dx;
    float B[3], Ex[3], Ey[3], Dg[3];  /* ortho (index space) */
    float Oe[3], F0[3];               /* persp: eye (index space), pixel-(0,0) world dir */
    float fwd[3];                     /* normalised forward, fp32 */
    float Ln[4][3];                   /* normalised to_light per light, fp32 */
    float Lg[4][3];                   /* to_light / dx per light, fp32 */
    float P[4];                       /* ortho phase per light, fp32 rounding of the fp64 value */
    double P64[4];                    /* the same in fp64 (used by the oracle's values) */
} orc_frame_constants;

typedef double (*orc_density_fn)(const float u[3], void* ctx);

double   orc_hg(double g, double cos_theta);
uint32_t orc_fmix32(uint32_t h);
uint32_t orc_jitter_hash(uint64_t seed, uint32_t frame_id, uint32_t pixel);
float    orc_jitter_delta(const orc_march* m, uint32_t frame_id, uint32_t pixel);
/* Trilinear border-zero sampler of C1 at padded index position u (fp32). */
double   orc_sample(const orc_grid* g, const float* vals, const float u[3]);

int orc_frame_constants_compute(const orc_grid* g, const orc_camera* cam,
                                const orc_light* lights, int32_t n_lights, int32_t light_mode,
                                const orc_medium* med, const orc_march* m,
                                orc_frame_constants* out);

/* One frame.  pix: NULL -> all W*H pixels in row-major order, else n_pix
 * pixel indices (py*W+px); outputs are indexed by position in that list.
 *   out_rgbt   n_pix*4 doubles  (L_r, L_g, L_b, T)
 *   out_depth  n_pix floats     (D, fp32 t value; 0 = no hit)
 *   out_debug  n_pix*6 u32 or NULL (n_lo, n_hi, n_hit, n_term, n_occ, light_samples)
 *   out_margin n_pix*2 doubles or NULL (depth-threshold margin, T_min margin; relative)
 *   forced_hit / forced_term: NULL or n_pix int32 (-1 = not forced)
 *   density_fn: NULL -> sample `vals`; else analytic density at padded index position
 *   no_clip_n: 0 -> conservative clip; >0 -> test every n in [1, no_clip_n] (pin P10)
 * Returns 0 on success, nonzero on invalid arguments. */
int orc_guiding_map(const orc_grid* g, const float* vals,
                    orc_density_fn density_fn, void* density_ctx,
                    const orc_camera* cam, const orc_light* lights, int32_t n_lights,
                    int32_t light_mode, const orc_medium* med, const orc_march* m,
                    uint32_t frame_id, int64_t n_pix, const int64_t* pix,
                    double* out_rgbt, float* out_depth, uint32_t* out_debug, double* out_margin,
                    const int32_t* forced_hit, const int32_t* forced_term, int32_t no_clip_n);

/* NEXT-4 transmittance-volume light model (V2-V5). */
typedef struct {
    double d[3], dhat[3], ell, e1[3], e2[3];   /* V2 (fp64) */
    int64_t a0, b0, k0, A, B, K;
} orc_tv_lattice;
/* V2 lattice of the light step vector d = hl * Lg (index units). */
int orc_tv_lattice_compute(const orc_grid* g, const float Lg[3], float hl, orc_tv_lattice* out);
/* V3/V4: tau_plus / tau_minus, A*B*K doubles each, index (j*K + k)*A + i... see orc_tv_index. */
int orc_tv_build(const orc_grid* g, const float* vals, orc_density_fn density_fn, void* density_ctx,
                 const orc_tv_lattice* lat, float hl, double kappa, double* tau_plus, double* tau_minus);
int64_t orc_tv_index(const orc_tv_lattice* lat, int64_t i, int64_t j, int64_t k);
/* V5 trilinear lookup of tau (either array) at index-space position U. */
double orc_tv_lookup(const orc_tv_lattice* lat, const double* tau, const float U[3]);
/* C8's optical depth kappa*hl*sum rho(U + j hl Lg) from U (the canonical light march). */
double orc_light_tau(const orc_grid* g, const float* vals, orc_density_fn density_fn, void* density_ctx,
                     const float U[3], const float Lg[3], float hl, double kappa);

/* NEXT-1 six-way bake (B1-B6). */
typedef struct {
    int32_t spp;                      /* samples per pixel >= 1 */
    float step, light_step;           /* h_b, h_bl (world units) */
    int32_t max_steps;                /* cap on k (0 = none) */
    float t_min;                      /* early termination (0 = off) */
    uint64_t seed;
} orc_bake;

void orc_bake_random(uint64_t seed, uint32_t frame, uint32_t pixel, uint32_t sample, float u_out[4]);
int orc_bake_light_constants(const orc_grid* g, const orc_camera* cam, float Lg[6][3], float Ln[6][3]);
/* out8: n_pix x 8 doubles in the Fig. 2 packing (right, top, back, T, left, bottom, front, E);
 * out_steps: NULL or n_pix u32 = in-support primary samples summed over the spp samples. */
int orc_sixway_bake(const orc_grid* g, const float* vals, orc_density_fn density_fn, void* density_ctx,
                    const orc_camera* cam, const orc_medium* med, const orc_bake* b, uint32_t frame_id,
                    int64_t n_pix, const int64_t* pix, double* out8, uint32_t* out_steps);

/* NEXT-2/3 relight + composite + depth shadow (R1-R3).
 * maps8: W*H*8 floats (Fig. 2 packing), depth: W*H floats or NULL; shadow_cams /
 * shadow_maps: NULL or per light (a NULL map = no shadow for that light);
 * out4: n_pix x 4 doubles (r, g, b, alpha); out_margin: NULL or n_pix doubles
 * (smallest shadow decision margin: pixel-boundary distance / relative depth gap). */
int orc_relight_weights(const orc_camera* cam, const orc_light* lights, int32_t n_lights, float c_out[][3]);
int orc_relight(const orc_camera* cam, const float* maps8, const float* depth, const orc_light* lights,
                int32_t n_lights, const float bg[3], const float emis[3], const orc_camera* shadow_cams,
                const float* const* shadow_maps, float bias, int64_t n_pix, const int64_t* pix, double* out4,
                double* out_margin);

#ifdef __cplusplus
}
#endif
#endif
