/* nsl_inputs/gen.c — seeded synthetic smoke volumes (test/bench INPUTS only).
 *
 * This module holds none of the guiding-map method's arithmetic: it only
 * manufactures density grids shaped like the paper's scenes (chimney/jet
 * plume P:151, obstacle-carved plume P:477 "cylindrical obstacles",
 * puff) so that the oracle (oracle/) and the CUDA path (paper_2604_03748_b200/)
 * can be fed identical, reproducible data.  The recipe is stated in DESIGN.md
 * §"Input recipe".  Both sides consume its output; neither is consulted here.
 *
 * Grid convention (DESIGN.md §Canonical C1): world box [0,1]^3, z up,
 * voxel (i,j,k) centred at ((i+.5)/n, (j+.5)/n, (k+.5)/n), values x-fastest,
 * fp32, values < 1e-6 flushed to 0 (no denormals), range [0,1].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

static uint32_t g_fmix32(uint32_t h) {
    h ^= h >> 16; h *= 0x85ebca6bu;
    h ^= h >> 13; h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

/* hash-lattice value in [0,1) */
static double lattice(int32_t x, int32_t y, int32_t z, uint32_t seed) {
    uint32_t h = g_fmix32((uint32_t)x * 0x8da6b343u ^ g_fmix32((uint32_t)y * 0xd8163841u ^
                 g_fmix32((uint32_t)z * 0xcb1ab31fu ^ seed)));
    return (double)(h >> 8) * (1.0 / 16777216.0);
}

static double smooth(double t) { return t * t * (3.0 - 2.0 * t); }

/* trilinear value noise with smoothstep weights */
static double vnoise(double x, double y, double z, uint32_t seed) {
    double fx = floor(x), fy = floor(y), fz = floor(z);
    int32_t ix = (int32_t)fx, iy = (int32_t)fy, iz = (int32_t)fz;
    double tx = smooth(x - fx), ty = smooth(y - fy), tz = smooth(z - fz);
    double c[2][2][2];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int d = 0; d < 2; ++d)
                c[a][b][d] = lattice(ix + d, iy + b, iz + a, seed);
    double x00 = c[0][0][0] + tx * (c[0][0][1] - c[0][0][0]);
    double x10 = c[0][1][0] + tx * (c[0][1][1] - c[0][1][0]);
    double x01 = c[1][0][0] + tx * (c[1][0][1] - c[1][0][0]);
    double x11 = c[1][1][0] + tx * (c[1][1][1] - c[1][1][0]);
    double y0 = x00 + ty * (x10 - x00);
    double y1 = x01 + ty * (x11 - x01);
    return y0 + tz * (y1 - y0);
}

/* 4-octave fBm, gain 0.5, normalised to [0,1) */
static double fbm(double x, double y, double z, uint32_t seed) {
    double s = 0.0, a = 1.0, norm = 0.0, f = 1.0;
    for (int o = 0; o < 4; ++o) {
        s += a * vnoise(x * f, y * f, z * f, seed + 0x9e37u * (uint32_t)o);
        norm += a; a *= 0.5; f *= 2.0;
    }
    return s / norm;
}

static double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

enum { KIND_PUFF = 0, KIND_PLUME = 1, KIND_CARVED = 2, KIND_CONST = 3 };

/* density at world point p for frame t; dx = voxel width (for the carved edge) */
static double density_at(int kind, double x, double y, double z, double t, double dx, uint32_t seed) {
    if (kind == KIND_CONST) return 1.0;
    if (kind == KIND_PUFF) {
        double r = sqrt((x - .5) * (x - .5) + (y - .5) * (y - .5) + (z - .5) * (z - .5));
        double base = 1.0 - r / 0.4;
        if (base <= 0.0) return 0.0;
        return clamp01(pow(base, 1.5) * (0.55 + 0.45 * fbm(8 * x, 8 * y, 8 * z, seed)));
    }
    /* plume / carved: inlet at z = 0.03, rising along +z, bent by a cross wind */
    if (z < 0.03) return 0.0;
    double zz = z - 0.03;
    double cx = 0.5 + 0.12 * zz * zz + 0.04 * sin(7.0 * zz - 0.05 * t), cy = 0.5 + 0.03 * cos(5.0 * zz - 0.03 * t);
    double obst = 1.0;
    if (kind == KIND_CARVED) {
        /* cylinder obstacle: axis y, centre (x=0.5, z=0.35), radius 0.08 */
        cx += 0.1 * exp(-((z - 0.35) / 0.12) * ((z - 0.35) / 0.12));
        double dcyl = sqrt((x - 0.5) * (x - 0.5) + (z - 0.35) * (z - 0.35)) - 0.08;
        obst = clamp01(dcyl / (2.0 * dx));
        if (obst <= 0.0) return 0.0;
    }
    /* turbulent radius: noise advected upward with the frame index */
    double nz_ = z - 0.004 * t;
    double turb = fbm(6 * x, 6 * y, 6 * nz_, seed);
    double R = (0.06 + 0.34 * zz) * (0.6 + 0.8 * turb);
    double r2 = ((x - cx) * (x - cx) + (y - cy) * (y - cy)) / (R * R);
    if (r2 >= 1.0) return 0.0;
    double prof = (1.0 - r2) * (1.0 - r2);
    double core = exp(-1.0 * zz);
    double detail = 0.2 + 0.8 * fbm(11 * x + 3.1, 11 * y + 1.7, 11 * nz_, seed ^ 0x51ed27u);
    double top = clamp01((0.97 - z) / 0.07);
    return clamp01(prof * core * detail * top * obst * 1.6);
}

typedef struct {
    int kind, nx, ny, nz, k0, k1;
    double t;
    uint32_t seed;
    float* out;
} job_t;

static void* run_job(void* arg) {
    job_t* j = (job_t*)arg;
    int nmax = j->nx > j->ny ? (j->nx > j->nz ? j->nx : j->nz) : (j->ny > j->nz ? j->ny : j->nz);
    double dx = 1.0 / (double)nmax;
    for (int k = j->k0; k < j->k1; ++k)
        for (int jj = 0; jj < j->ny; ++jj)
            for (int i = 0; i < j->nx; ++i) {
                double v = density_at(j->kind, (i + 0.5) * dx, (jj + 0.5) * dx, (k + 0.5) * dx, j->t, dx, j->seed);
                float f = (float)v;
                if (!(f >= 1e-6f)) f = 0.0f;
                j->out[((size_t)k * j->ny + jj) * j->nx + i] = f;
            }
    return NULL;
}

/* Fill out[nz][ny][nx] (x-fastest).  Returns 0 on success.  Deterministic for
 * fixed (kind, dims, t, seed) irrespective of n_threads (disjoint z slabs). */
int nslgen_volume(int kind, int nx, int ny, int nz, double t, uint32_t seed, int n_threads, float* out) {
    if (kind < 0 || kind > KIND_CONST || nx < 1 || ny < 1 || nz < 1 || !out) return 1;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_threads > nz) n_threads = nz;
    pthread_t th[256];
    job_t jobs[256];
    for (int p = 0; p < n_threads; ++p) {
        jobs[p] = (job_t){kind, nx, ny, nz, (int)((long)nz * p / n_threads), (int)((long)nz * (p + 1) / n_threads), t, seed, out};
        if (n_threads == 1) run_job(&jobs[p]);
        else pthread_create(&th[p], NULL, run_job, &jobs[p]);
    }
    if (n_threads > 1)
        for (int p = 0; p < n_threads; ++p) pthread_join(th[p], NULL);
    return 0;
}

/* FNV-1a 64 over the raw bytes (content hash recorded with each workload). */
uint64_t nslgen_fnv1a64(const void* data, size_t n) {
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) { h ^= p[i]; h *= 0x100000001b3ull; }
    return h;
}
