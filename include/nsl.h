/* include/nsl.h — C ABI of the B200-native guiding-map ray march.
 *
 * Operation: Algorithm 1 of "Real-time Neural Six-way Lightmaps"
 * (arXiv 2604.03748; "Ray-marching for Guiding Map
 * L~_scattering"), with h = 10 dx on sigma_s "in a 3D texture" (L410) and
 * the surrogate lights front = omega, top = omega x z, bottom = -omega x z of
 * eq:approx (L361-365).  The precise canonical definition (C1-C14) that the
 * kernels implement is DESIGN.md §2; each entry point below cites it.
 *
 * Conventions shared by every entry point
 *   - Plain C; every function returns nsl_status and never aborts/throws.
 *     On failure nsl_last_error() returns a thread-local message.
 *   - Arguments are validated on the host BEFORE anything is enqueued;
 *     invalid input -> NSL_ERR_INVALID_ARG, nothing enqueued.
 *   - Device pointers are plain CUDA device addresses (e.g. torch tensors'
 *     data_ptr()); `stream` is a cudaStream_t (nsl_stream is ABI-identical).
 *     All device work is enqueued asynchronously on `stream`; asynchronous
 *     device faults surface at the caller's next synchronisation.
 *   - Host structs are read only during the call and never retained.
 *   - Output buffers are caller-owned; the library never allocates outputs.
 *     Transient per-call workspaces (frame tables) are taken from the
 *     device's stream-ordered pool (cudaMallocAsync) and freed on `stream`.
 *   - The current CUDA device is used; buffers must live on it.
 */
#ifndef NSL_H
#define NSL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* nsl_stream;          /* == cudaStream_t */

typedef enum {
    NSL_OK = 0,
    NSL_ERR_INVALID_ARG = 1,
    NSL_ERR_UNSUPPORTED = 2,
    NSL_ERR_OUT_OF_MEMORY = 3,
    NSL_ERR_CUDA = 4
} nsl_status;

/* Thread-local text of the last non-OK status ("" if none). */
const char* nsl_last_error(void);
/* Library version string (static storage). */
const char* nsl_version(void);

/* ------------------------------------------------------------------ volume (row a1)
 * Density grid sigma_s carrier ("smoke data sigma_s in a 3D
 * texture"; C1): nx*ny*nz finite values >= 0,
 * x-fastest, voxel (i,j,k) centred at origin + (i+.5, j+.5, k+.5)*voxel_width.
 * Requires nx,ny,nz >= 1, voxel_width > 0, (nx+2)(ny+2)(nz+2) < 2^31. */
typedef struct {
    int32_t nx, ny, nz;
    float origin[3];
    float voxel_width;
} nsl_grid_desc;

/* Device layouts.  All carry the 1-voxel zero apron of C1.
 *  LINEAR_F32 : (nx+2)(ny+2)(nz+2) floats, x-fastest (8 scalar gathers/sample)
 *  QUAD_F32   : per padded cell (i,j,k), i<=nx, j<=ny, k<=nz+1, a float4 of the
 *               x/y 2x2 corner quad (2 x 16-B gathers/sample), exact fp32 values
 *  CORNER_F16 : per padded cell (i,j,k), i<=nx, j<=ny, k<=nz, all 8 corners as
 *               fp16 (1 x 16-B gather/sample); values rounded RNE to fp16
 *  OCT_F32    : per padded cell (i,j,k), i<=nx, j<=ny, k<=nz, the QUAD float4 of
 *               planes k and k+1 side by side (32 B: one 256-bit gather/sample),
 *               exact fp32 values; storage must be 32-B aligned.  With 4^3 / 8^3
 *               occupancy blocks (grids up to ~640^3) only the elements of occupied
 *               blocks are written -- the march never reads the others -- so the
 *               bytes of empty blocks keep whatever the storage held before
 *  BRICK_OCT_F32: the OCT elements in 4x4x4-cell bricks (2 KB each, x fastest inside
 *               a brick): one 256-bit gather/sample, 3-D locality per 128-B line;
 *               storage must be 32-B aligned.  Measured against OCT: the
 *               better choice for a static volume far beyond L2 (512^3, 4.3 GB: C5 march
 *               -5 % over 1024 frames, -11 % over 64), worse at 256^3 (C3 +2 %) and for
 *               a fresh volume per frame (its build costs 2x).
 *  TEX3D_F32  : the QUAD float4 of every padded cell in a LIBRARY-OWNED 3-D cudaArray read
 *               through a point-sampled texture object (2 tex fetches/sample, hardware
 *               3-D addressing, block-linear tiling); `device_storage` holds only the
 *               occupancy region and tail (nsl_volume_bytes says how much).  Exact fp32
 *               values (hardware trilinear FILTERING is not used: its 8-bit fractional
 *               weights cannot meet the 1e-4 bar).  nsl_volume_release frees
 *               the array; nsl_volume_rebuild refills it in place.
 *  MORTON_OCT_F32: the OCT elements in 8x8x8-cell tiles (16 KB, tiles x-fastest), Morton
 *               (z-order) inside a tile; one 256-bit gather/sample; 32-B aligned storage.
 *  AUTO       : chosen from the grid size (nsl_layout_resolve).  DEFAULT = AUTO. */
typedef enum {
    NSL_LAYOUT_LINEAR_F32 = 0,
    NSL_LAYOUT_QUAD_F32 = 1,
    NSL_LAYOUT_CORNER_F16 = 2,
    NSL_LAYOUT_OCT_F32 = 3,
    NSL_LAYOUT_BRICK_OCT_F32 = 4,
    NSL_LAYOUT_TEX3D_F32 = 5,
    NSL_LAYOUT_MORTON_OCT_F32 = 6,
    NSL_LAYOUT_AUTO = 7,
    NSL_LAYOUT_DEFAULT = NSL_LAYOUT_AUTO
} nsl_layout;

/* The concrete layout NSL_LAYOUT_AUTO stands for on grid g (any other layout is returned as
 * is; -1 on an invalid grid): BRICK_OCT_F32 when the OCT body (n_x+1)(n_y+1)(n_z+1) x 32 B
 * exceeds 2 GiB, else OCT_F32 -- chosen by measurement.  Every entry point
 * taking a layout resolves AUTO this way (nsl_guiding_map_animated: OCT_F32, since its
 * per-frame builds favour the cheaper OCT build). */
int32_t nsl_layout_resolve(const nsl_grid_desc* g, int32_t layout);

/* Kernel launches one volume build (nsl_volume_upload / nsl_volume_rebuild) enqueues for grid g
 * and layout (AUTO resolved): 3 for OCT_F32 with 4^3 / 8^3 occupancy blocks (occupancy reset,
 * staged occupancy-gated layout, finalize), else 2 (fused layout + occupancy, finalize).
 * -1 on an invalid grid or layout.  For launch accounting and graph sizing. */
int32_t nsl_volume_build_launches(const nsl_grid_desc* g, int32_t layout);

typedef struct nsl_volume nsl_volume;             /* opaque, immutable after upload */

/* Device bytes the caller must provide as `device_storage` for `layout`
 * (0 on invalid arguments). */
size_t nsl_volume_bytes(const nsl_grid_desc* g, int32_t layout);

/* Build the device layout from `density` (x-fastest nx*ny*nz floats) into the
 * caller-owned `device_storage` (>= nsl_volume_bytes, 16-B aligned) on
 * `stream`, and return a handle in *out.
 *   density_on_device = 0: `density` is host memory (pinned or pageable);
 *     values are validated on the host (finite, >= 0) before enqueueing.
 *   density_on_device = 1: `density` is device memory; values are checked by
 *     the layout kernel, and nsl_volume_check() reports the result.
 * Host input: the call returns once the host->device copy of `density` has
 * completed (it waits for the copy, not for the layout build), so the host
 * buffer -- pinned or pageable -- may be refilled or freed on return.
 * The handle does not own `device_storage`; the storage (and, for host
 * input, nothing else) must outlive every call that reads the volume. */
nsl_status nsl_volume_upload(const nsl_grid_desc* g, const float* density, int32_t density_on_device,
                             int32_t layout, void* device_storage, size_t storage_bytes,
                             nsl_stream stream, nsl_volume** out);
/* Synchronises `stream` and reports whether the layout kernel saw a
 * non-finite or negative input value (*n_invalid = count). */
nsl_status nsl_volume_check(const nsl_volume* v, nsl_stream stream, uint64_t* n_invalid);
/* Frees the handle (never the caller's storage).  NULL is a no-op. */
nsl_status nsl_volume_release(nsl_volume* v);
/* Rebuild an existing handle's layout in place from new density values (same grid, layout and
 * storage; TEX3D: the same array), e.g. a simulator streaming one frame after another into one
 * volume slot.  Host / device density and validation exactly as
 * nsl_volume_upload; plans referencing the volume see the new values.  Asynchronous on
 * `stream` (host input: returns once the density has been copied). */
nsl_status nsl_volume_rebuild(nsl_volume* v, const float* density, int32_t density_on_device, nsl_stream stream);

/* ------------------------------------------------------------------ frame parameters
 * Camera (C3).  forward and up must be finite,
 * |forward| within 1e-3 of 1 (renormalised), up not parallel to forward.
 *   projection 0 = orthographic (billboard, canonical), 1 = perspective;
 *   extent: ortho image-plane height (world units, > 0); persp 2*tan(fov_y/2).
 *   position: ortho image-plane centre; persp eye. */
typedef struct {
    int32_t projection;
    float position[3], forward[3], up[3];
    float extent;
    int32_t width, height;
} nsl_camera;

/* Directional light (eq:approx L_s): to_light unit (scene -> light,
 * |.| within 1e-3 of 1), rgb radiance >= 0.  In guide mode to_light is
 * ignored and derived from the camera (C3b). */
typedef struct {
    float to_light[3];
    float rgb[3];
} nsl_light;

enum { NSL_LIGHTS_EXPLICIT = 0, NSL_LIGHTS_GUIDE = 1 };
enum { NSL_OPACITY_EXP = 0, NSL_OPACITY_RIEMANN = 1, NSL_OPACITY_LITERAL = 2 };

/* Medium (C2): sigma_t = extinction*rho, sigma_s = albedo*sigma_t;
 * extinction >= 0, albedo in [0,1], hg_g in (-1,1) (HG phase). */
typedef struct {
    float extinction, albedo, hg_g;
} nsl_medium;

/* March parameters (Alg. 1 inputs "step size h, number of steps N", P:374;
 * DESIGN.md C4-C13).  step > 0 (paper: 10*voxel_width); light_step
 * >= 0 (0 -> step); max_steps >= 0 (0 -> to the support exit); depth_tau >= 0
 * compared with sigma_s; t_min in [0,1) (0 = no early termination);
 * opacity_form NSL_OPACITY_*; jitter 0/1; guide_axis: the world "z" of
 * omega x z ((0,0,0) -> (0,0,1)); front_identity 0/1 allows the C9 shortcut;
 * light_model NSL_LIGHT_MARCH (C8, canonical) or NSL_LIGHT_TV (NEXT-4,
 * per frame and light a swept optical-depth lattice, one
 * interpolated lookup per occupied sample; frames are processed in groups
 * whose lattices fit NSL_TV_BUDGET_MB (default 4096) of transient device memory). */
enum { NSL_LIGHT_MARCH = 0, NSL_LIGHT_TV = 1 };
typedef struct {
    float step, light_step;
    int32_t max_steps;
    float depth_tau, t_min;
    int32_t opacity_form;
    int32_t jitter;
    uint64_t seed;
    float guide_axis[3];
    int32_t front_identity;
    int32_t light_model;
} nsl_march;

/* ------------------------------------------------------------------ the march (rows a2-a8)
 * One frame of Algorithm 1 for every pixel of cam (C3-C12).
 *   lights: n_lights (1..4) entries; light_mode NSL_LIGHTS_* (guide: n_lights <= 3).
 *   frame_id: jitter key (C4).
 *   out_rgbt:  device, H*W float4 (L_r, L_g, L_b, T), row-major, row 0 = top, 16-B aligned
 *   out_depth: device, H*W floats (D; 0 = no hit)
 *   out_debug: device, H*W*6 u32 (n_lo, n_hi, n_hit, n_term, n_occ, light_samples) or NULL;
 *              when non-NULL the C9 shortcut is disabled (counters are the canonical ones). */
nsl_status nsl_guiding_map(const nsl_volume* vol, const nsl_camera* cam,
                           const nsl_light* lights, int32_t n_lights, int32_t light_mode,
                           const nsl_medium* med, const nsl_march* m, uint32_t frame_id,
                           float* out_rgbt, float* out_depth, uint32_t* out_debug,
                           nsl_stream stream);

/* A batch of F independent frames in ONE launch (row a9; frames are
 * independent, "streamed directly into the guiding map generation").
 *   vols[n_vols]; frame_vol[F] indexes vols; cams[F] (all the same W, H);
 *   lights[F*n_lights]; frame_ids[F] jitter keys (global frame ids, so that
 *   sharded runs equal the unsharded one bit for bit).
 *   out_rgbt F*H*W float4, out_depth F*H*W floats, out_debug F*H*W*6 u32 or NULL. */
nsl_status nsl_guiding_map_batch(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                                 const nsl_camera* cams, const nsl_light* lights, int32_t n_lights,
                                 int32_t light_mode, const nsl_medium* med, const nsl_march* m,
                                 const uint32_t* frame_ids, int32_t F,
                                 float* out_rgbt, float* out_depth, uint32_t* out_debug,
                                 nsl_stream stream);

/* The same launch as nsl_guiding_map_batch (identical results, the timed
 * fast path), instrumented: it also accumulates into `counters` (device,
 * 8 x u64, zeroed by the call on `stream`):
 *   [0] primary samples processed  = sum over pixels of (n_term - n_lo + 1)
 *   [1] light samples (canonical)  = sum over pixels of light_samples (C12)
 *   [2] trilinear gathers executed (samples in non-empty occupancy blocks that
 *       the kernel actually loaded; the C9 front march is not executed)
 *   [3] occupied primary samples   = sum of n_occ
 *   [4] primary samples tested (occupied-box sub-range actually walked)
 *   [5] light samples tested (occupied-box-clipped marches actually walked)
 *   [6], [7] reserved (0)
 * [0]+[1] is the canonical march-sample count of DESIGN.md §7. */
nsl_status nsl_guiding_map_batch_counted(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                                         const nsl_camera* cams, const nsl_light* lights, int32_t n_lights,
                                         int32_t light_mode, const nsl_medium* med, const nsl_march* m,
                                         const uint32_t* frame_ids, int32_t F,
                                         float* out_rgbt, float* out_depth, uint64_t* counters,
                                         nsl_stream stream);

/* Plans: the same batch, prepared once.  nsl_plan_create validates and
 * marshals the per-frame inputs (cameras, lights, frame ids, volume
 * references) exactly as nsl_guiding_map_batch does and uploads them into
 * plan-owned device memory (cudaMalloc; the upload is enqueued on `stream`).
 * nsl_plan_execute then enqueues only device work — the per-frame setup
 * kernel (rows a2/a3) and the march kernel (rows a4-a8) — with no host
 * marshalling and no host<->device copy, so it is cheap to call every frame
 * and capturable in a CUDA graph.  Results are identical to the batch call.
 * The referenced volumes' device storage must stay valid (re-uploading a
 * volume into the same storage between executions is allowed: the plan keeps
 * the storage pointers, not the host handles).  out_debug / counters as in
 * nsl_guiding_map_batch / _counted (at most one of them non-NULL).
 * nsl_plan_destroy frees the plan's device memory (synchronising the device).
 * Concurrency: a plan owns one device workspace (per-frame parameters, tile
 * cull flags, TV lattices) that every execution rewrites, so executions of
 * ONE plan must be ordered -- the same stream, or streams/graphs ordered by
 * events; never two in flight at once.  Independent plans may run
 * concurrently. */
typedef struct nsl_plan nsl_plan;
nsl_status nsl_plan_create(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                           const nsl_camera* cams, const nsl_light* lights, int32_t n_lights,
                           int32_t light_mode, const nsl_medium* med, const nsl_march* m,
                           const uint32_t* frame_ids, int32_t F, nsl_stream stream, nsl_plan** out);
nsl_status nsl_plan_execute(const nsl_plan* plan, float* out_rgbt, float* out_depth, uint32_t* out_debug,
                            uint64_t* counters, nsl_stream stream);
nsl_status nsl_plan_destroy(nsl_plan* plan);

/* ------------------------------------------------------------------ NEXT-1: six-way bake
 * Reference single-scatter six-way lightmaps (B1-B6): the
 * lightmaps {L_x^+-, L_y^+-, L_z^+-} along the camera's billboard axes
 * (PAPER.md L219), transparency (L255) and an emissive carrier, by jittered
 * fixed-step quadrature with `spp` counter-based samples per pixel (L477
 * "single bounce ... g = 0 ... samples per pixel").  Volumes, cameras and
 * medium as for nsl_guiding_map_batch (lights are fixed: six unit-white
 * axis lights).  spp >= 1; step > 0 (h_b), light_step > 0 (h_bl); max_steps
 * >= 0 caps k; t_min in [0,1).
 *   out: device, F*H*W*8 floats = two float4 per pixel in the Fig. 2 packing:
 *        (right +X, top +Y, back -Z, transparency) (left -X, bottom -Y, front +Z, emissive)
 *   counters: device u64[1] (zeroed by the call) += trilinear gathers, or NULL. */
typedef struct {
    int32_t spp;
    float step, light_step;
    int32_t max_steps;
    float t_min;
    uint64_t seed;
} nsl_bake;

nsl_status nsl_sixway_bake(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                           const nsl_camera* cams, const nsl_medium* med, const nsl_bake* b,
                           const uint32_t* frame_ids, int32_t F, float* out, uint64_t* counters,
                           nsl_stream stream);

/* The six bake light directions as the device computes them (fp64 -> fp32):
 * Lg[l] = n_l / dx, Ln[l] = n_l in the B6 order (right, top, back, left,
 * bottom, front); host outputs; synchronises `stream`. */
nsl_status nsl_debug_bake_lights(const nsl_grid_desc* g, const nsl_camera* cam, float Lg[6][3], float Ln[6][3],
                                 nsl_stream stream);

/* ------------------------------------------------------------------ NEXT-2/3: relight + shadow
 * Six-way relighting, composite and depth-based obstacle shadow (DESIGN.md
 * §11, R1-R3): per pixel out = sum_l rgb_l * v_l * sum_p |c_p| L_p^sign(c_p)
 * + emis * E + T * bg, alpha = 1 - T (Fig. 2 packing),
 * with v_l the shadow visibility of the smoke shell (guiding-map depth D)
 * against light l's orthographic shadow map (L458-462).
 *   cams[F] (same W, H); maps: device F*H*W*8 floats (Fig. 2 packing);
 *   depth: device F*H*W floats or NULL (no shadows); lights[F*n_lights]
 *   (1..4, unit to_light); bg[3], emis[3] host; shadow_cams: host F*n_lights
 *   cameras (projection 0, looking along -to_light) or NULL; shadow_maps:
 *   host array of F*n_lights DEVICE pointers (Hs*Ws floats, world depth along
 *   the shadow camera's forward, +inf = empty) with NULL entries allowed, or
 *   NULL; bias >= 0.  out: device F*H*W float4 (r, g, b, alpha). */
nsl_status nsl_relight(const nsl_camera* cams, int32_t F, const float* maps, const float* depth,
                       const nsl_light* lights, int32_t n_lights, const float bg[3], const float emis[3],
                       const nsl_camera* shadow_cams, const float* const* shadow_maps, float bias,
                       float* out, nsl_stream stream);

/* End-to-end convenience call with HOST buffers: uploads the host density
 * grid, lays it out, marches the F frames and copies the results back into
 * host out_rgbt (F*H*W*4 floats) / out_depth (F*H*W floats); synchronises
 * `stream` before returning.  The frames are marched in chunks on `stream`
 * while the previous chunk's results stream back on an internal side stream.
 * The density is validated on the device (the build kernel's count): a
 * non-finite or negative value makes the call return NSL_ERR_INVALID_ARG
 * (the host outputs are then unspecified).  All device memory is transient
 * (stream-ordered pool).  Host buffers may be pageable; pinned memory makes
 * the copies asynchronous DMA. */
nsl_status nsl_guiding_map_host(const nsl_grid_desc* g, const float* host_density, int32_t layout,
                                const nsl_camera* cams, const nsl_light* lights, int32_t n_lights,
                                int32_t light_mode, const nsl_medium* med, const nsl_march* m,
                                const uint32_t* frame_ids, int32_t F,
                                float* host_rgbt, float* host_depth, nsl_stream stream);
/* The same with a compact download: the fp32 maps are rounded to IEEE binary16 (RNE) on the
 * device and host_rgbt_h (F*H*W*4 halves) / host_depth_h (F*H*W halves) receive 10 B per
 * pixel instead of 20 -- half the PCIe traffic that bounds the host call.  The march and its
 * fp32 results are unchanged; only the delivered values are rounded (relative error <= 2^-11,
 * so this output is NOT the 1e-4 parity path: use nsl_guiding_map_host for that). */
nsl_status nsl_guiding_map_host_f16(const nsl_grid_desc* g, const float* host_density, int32_t layout,
                                    const nsl_camera* cams, const nsl_light* lights, int32_t n_lights,
                                    int32_t light_mode, const nsl_medium* med, const nsl_march* m,
                                    const uint32_t* frame_ids, int32_t F, uint16_t* host_rgbt_h,
                                    uint16_t* host_depth_h, nsl_stream stream);

/* Animated volumes (SURVEY §8(a) rows a1 + a9, config C4; the simulator's
 * density is "streamed directly into the guiding map generation", one grid per frame).
 * Frame f's density densities[f] (DEVICE pointer, x-fastest nx*ny*nz fp32, like
 * nsl_volume_upload with density_on_device = 1) is laid out into storage[f] (caller-owned
 * device memory of storage_bytes >= nsl_volume_bytes(g, layout), aligned as for
 * nsl_volume_upload; one buffer per frame, not shared between frames) and marched with
 * cams[f] and lights[f*n_lights ...].  densities and storage are HOST arrays of F device
 * pointers.  Frames run in chunks of `chunk` frames (0 -> 6): the layouts of chunk c+1 build
 * on an internal side stream while chunk c marches on `stream` (results of early chunks are
 * ready early; how much of the HBM-bound build hides under the march depends on the march's
 * length).  Results are bitwise those of nsl_volume_upload of every
 * frame followed by nsl_guiding_map_batch; outputs as nsl_guiding_map_batch (device, F*H*W*4
 * and F*H*W floats).  Asynchronous: all work is ordered on `stream` on return, unless
 * n_invalid (host pointer) is non-NULL, in which case the call synchronises `stream` and
 * stores the number of non-finite or negative density values over all frames (counted by
 * the build kernels; the maps of such frames are unspecified). */
nsl_status nsl_guiding_map_animated(const nsl_grid_desc* g, const float* const* densities, int32_t layout,
                                    void* const* storage, size_t storage_bytes, const nsl_camera* cams,
                                    const nsl_light* lights, int32_t n_lights, int32_t light_mode,
                                    const nsl_medium* med, const nsl_march* m, const uint32_t* frame_ids,
                                    int32_t F, int32_t chunk, float* out_rgbt, float* out_depth,
                                    uint64_t* n_invalid, nsl_stream stream);

/* The surrogate light set of eq:approx (C3b) for a camera:
 * out[0] front = omega = -forward, out[1] top = normalize(omega x axis), out[2] bottom =
 * -top (axis NULL -> world z; fallback x^ when omega is parallel to axis), as the fp32 unit
 * vectors the march uses in NSL_LIGHTS_GUIDE mode (computed by the same device code), each
 * with radiance rgb (NULL -> white).  Host outputs; synchronises `stream`. */
nsl_status nsl_guide_lights(const nsl_camera* cam, const float axis[3], const float rgb[3], nsl_light out[3],
                            nsl_stream stream);

/* Sampler microbenchmark (SURVEY §8(d) "Denominators"): the march's own light-sample loop
 * (sampler.cuh light_sum: positions, occupancy test, one gather, trilinear) run by every
 * thread of waves x (SMs x resident CTAs) CTAs of 128 threads over 16-sample lines inside
 * [2, 15)^3 of `vol` (>= 16^3; meant for a small, fully occupied, L1-resident grid), reps
 * times; warps on the march's 8 x 4 footprint at a 0.25-voxel pixel pitch.  sink: device,
 * >= threads floats (written, keeps the work live).  *samples (host) = samples the launch
 * takes; time it with events on `stream`.  Asynchronous. */
nsl_status nsl_bench_l1_gather(const nsl_volume* vol, int32_t waves, int32_t reps, float* sink, size_t sink_floats,
                               uint64_t* samples, nsl_stream stream);

/* Hardware L1/TEX gather ceiling (the roofline denominator of the march): every
 * lane of waves x (SMs x resident CTAs) CTAs of 256 threads issues reps x 16 loads of one
 * 32-B element (ld.global.nc.v8.f32, the OCT sampler's gather) at element offsets
 * lane_off[k*32 + lane] (k = 0..15; device int32[512], each in [0, max_off]) from
 * buf + 32 B * shift_r, shift_r = (r * stride_elems) mod span_elems, and sums the eight
 * floats -- no other work.  stride_elems = 0: every load hits the same few L1-resident
 * lines (the L1 ceiling for that lane pattern).  buf: device, 32-B aligned, >= (span_elems +
 * max_off) * 8 floats; sink: device, >= threads floats.  *bytes (host) = lane bytes the
 * launch loads (threads * reps * 16 * 32).  Time it with events on `stream`.  Asynchronous. */
nsl_status nsl_bench_l1_peak(const float* buf, size_t buf_floats, const int32_t* lane_off, int32_t max_off,
                             int64_t stride_elems, int64_t span_elems, int32_t waves, int32_t reps, float* sink,
                             size_t sink_floats, uint64_t* bytes, nsl_stream stream);

/* The paper's "3D texture" sampling with HARDWARE trilinear filtering, for measuring
 * its precision against the canonical fp32 sampler: the padded grid of
 * `density` (device, x-fastest) in a float cudaArray with cudaFilterModeLinear and border
 * (zero) addressing, sampled at n padded-index positions (device float[3n]) into out (device
 * float[n]).  Synchronous; allocates and frees its own array. */
nsl_status nsl_debug_tex_filter(const nsl_grid_desc* g, const float* density, const float* positions, int32_t n,
                                float* out, nsl_stream stream);

/* ------------------------------------------------------------------ debug / verification
 * Frame constants of DESIGN.md C3/C3b/C10 as the device computes them
 * (fp64 evaluation rounded once to fp32), for bitwise comparison with the
 * oracle (pin P15).  Synchronises `stream`; `out` is host memory. */
typedef struct {
    float inv_dx;
    float B[3], Ex[3], Ey[3], Dg[3];
    float Oe[3], F0[3];
    float fwd[3];
    float Ln[4][3];
    float Lg[4][3];
    float P[4];
    int32_t front_identity_ok;
} nsl_frame_constants;

nsl_status nsl_debug_frame_constants(const nsl_grid_desc* g, const nsl_camera* cam,
                                     const nsl_light* lights, int32_t n_lights, int32_t light_mode,
                                     const nsl_medium* med, const nsl_march* m,
                                     nsl_frame_constants* out, nsl_stream stream);

/* The C4 jitter chain on the device: for pixels 0..n-1 of a row-major
 * image, out_hash[p] = h32, out_delta[p] = delta (device buffers). */
nsl_status nsl_debug_jitter(const nsl_march* m, uint32_t frame_id, int32_t n,
                            uint32_t* out_hash, float* out_delta, nsl_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* NSL_H */
