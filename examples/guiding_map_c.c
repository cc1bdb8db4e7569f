/* examples/guiding_map_c.c — the C ABI from plain C (no CUDA headers, no Python):
 * a procedural smoke ball, the paper's guide lights (front, top, bottom; PAPER.md
 * L361-365) and large step h = 10 dx (L410), marched for a few orbiting frames through
 * nsl_guiding_map_host (host buffers in and out), then a few sanity checks.
 *
 *   gcc -std=c99 -O2 -Iinclude examples/guiding_map_c.c \
 *       -Lpaper_2604_03748_b200/lib -lnsl -Wl,-rpath,$PWD/paper_2604_03748_b200/lib -lm -o /tmp/gm
 *   /tmp/gm        # prints per-frame coverage / mean transmittance / max scattering; exit 0 = ok
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "nsl.h"

#define N 64
#define RES 128
#define FRAMES 4

int main(void) {
    printf("%s\n", nsl_version());
    nsl_grid_desc g = {N, N, N, {0.0f, 0.0f, 0.0f}, 1.0f / N};
    float* dens = (float*)malloc(sizeof(float) * N * N * N);
    for (int k = 0; k < N; ++k)                  /* a soft ball of radius 0.3 in the unit box */
        for (int j = 0; j < N; ++j)
            for (int i = 0; i < N; ++i) {
                const float x = (i + 0.5f) / N - 0.5f, y = (j + 0.5f) / N - 0.5f, z = (k + 0.5f) / N - 0.5f;
                const float r = sqrtf(x * x + y * y + z * z);
                dens[(k * N + j) * N + i] = r < 0.3f ? 1.0f - r / 0.3f : 0.0f;
            }
    nsl_camera cams[FRAMES];
    nsl_light lights[FRAMES * 3];
    uint32_t ids[FRAMES];
    for (int f = 0; f < FRAMES; ++f) {           /* orthographic billboard cameras orbiting z */
        const float a = 0.5f * f, c = cosf(a), s = sinf(a);
        nsl_camera cam = {0, {0.5f + 2.0f * c, 0.5f + 2.0f * s, 0.5f}, {-c, -s, 0.0f}, {0.0f, 0.0f, 1.0f},
                          1.2f, RES, RES};
        cams[f] = cam;
        for (int l = 0; l < 3; ++l) {            /* guide mode: directions ignored, colours used */
            nsl_light L = {{1.0f, 0.0f, 0.0f}, {1.0f, 1.0f, 1.0f}};
            lights[f * 3 + l] = L;
        }
        ids[f] = (uint32_t)f;
    }
    nsl_medium med = {32.0f, 0.9f, 0.0f};
    nsl_march m = {10.0f / N, 0.0f, 0, 0.3f, 1e-4f, NSL_OPACITY_EXP, 1, 0x6B616B65ull, {0.0f, 0.0f, 1.0f}, 1,
                   NSL_LIGHT_MARCH};
    float* rgbt = (float*)malloc(sizeof(float) * 4 * RES * RES * FRAMES);
    float* depth = (float*)malloc(sizeof(float) * RES * RES * FRAMES);
    nsl_status st = nsl_guiding_map_host(&g, dens, NSL_LAYOUT_DEFAULT, cams, lights, 3, NSL_LIGHTS_GUIDE, &med, &m,
                                         ids, FRAMES, rgbt, depth, NULL);
    if (st != NSL_OK) {
        fprintf(stderr, "nsl_guiding_map_host: %s\n", nsl_last_error());
        return 1;
    }
    int ok = 1;
    for (int f = 0; f < FRAMES; ++f) {
        double tsum = 0.0, lmax = 0.0;
        int covered = 0;
        for (int p = 0; p < RES * RES; ++p) {
            const float* o = rgbt + 4 * ((size_t)f * RES * RES + p);
            tsum += o[3];
            if (o[0] > lmax) lmax = o[0];
            covered += depth[(size_t)f * RES * RES + p] > 0.0f;
            if (!(o[3] >= 0.0f && o[3] <= 1.0f) || !(o[0] >= 0.0f)) ok = 0;
        }
        /* the ball covers pi 0.3^2 / 1.2^2 ~ 20 % of the image; the centre ray is opaque */
        const float tc = rgbt[4 * ((size_t)f * RES * RES + (RES / 2) * RES + RES / 2) + 3];
        printf("frame %d: covered %.3f  mean T %.3f  centre T %.2e  max L %.4f\n", f, covered / (double)(RES * RES),
               tsum / (RES * RES), tc, lmax);
        if (covered < RES * RES / 10 || covered > RES * RES / 3 || tc > 1e-3f || lmax <= 0.0) ok = 0;
    }
    /* invalid input is rejected before anything runs */
    dens[7] = -1.0f;
    if (nsl_guiding_map_host(&g, dens, NSL_LAYOUT_DEFAULT, cams, lights, 3, NSL_LIGHTS_GUIDE, &med, &m, ids, FRAMES,
                             rgbt, depth, NULL) != NSL_ERR_INVALID_ARG)
        ok = 0;
    free(dens);
    free(rgbt);
    free(depth);
    printf(ok ? "ok\n" : "FAILED\n");
    return ok ? 0 : 1;
}
