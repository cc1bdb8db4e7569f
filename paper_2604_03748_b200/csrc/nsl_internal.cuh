// nsl_internal.cuh — device-side types of libnsl (B200 guiding-map ray march).
// Not part of the ABI.  See include/nsl.h for the boundary and DESIGN.md §2
// for the canonical definition every kernel follows.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/nsl.h"

namespace nsl {

// Occupancy bitmask geometry (DESIGN.md §6 "empty-space skip"): one bit per
// block of (2^shift)^3 padded cells; cell c = floor(U) in [0, n] per axis.
// A clear bit means every corner of every cell of the block is 0, so any
// trilinear sample whose cell lies in the block is exactly 0 (C1).
struct OccGeom {
    int32_t shift, nbx, nby, nbz;
    int32_t words;             // ceil(nbx*nby*nbz / 32), padded to a multiple of 4
    int32_t words_total;       // mask + per-slab boxes: words + 4*nbz (a multiple of 4)
    int32_t rowwords, rows;    // build scratch: per block row (by, bz) ceil(nbx/32) flag words, then
    int32_t info_off;          // at word info_off (a multiple of 4) a 4-word record per row
    int32_t scratch_words;     // (min bx, max bx, invalid voxels, -)
};
// Occupancy region (device, staged to shared memory by the march):
//   [mask: words u32][slab_min: nbz x (bx, by) int32][slab_max: nbz x (bx, by) int32]
// slab box of z-block slab bz = the x/y range of its non-empty blocks (min > max: empty).
OccGeom occ_geom(int nx, int ny, int nz);
// OCT volumes with 4^3 / 8^3 occupancy blocks build through the staged, occupancy-gated kernel
// (3 launches: occ_reset, oct_build, occ_finalize); every other layout through the fused one (2)
bool staged_oct_build(int layout, const OccGeom& g);

// Per-volume description handed to the frame-setup kernel.
struct VolDesc {
    const void* data;
    int32_t nx, ny, nz, layout;
    float origin[3];
    float dx;
    const uint32_t* occ;
    OccGeom og;
    const int32_t* aabb;       // occupied block bounds: bmin xyz, bmax xyz (bmin > bmax: empty volume)
    unsigned long long surf;   // TEX3D: surface object of the library-owned array (the build writes it)
};

// Raw per-frame input (host -> device, one memcpy per call).
struct FrameIn {
    nsl_camera cam;
    VolDesc vol;
    uint32_t frame_id;
    int32_t pad;
};

// Per-frame constants produced by frame_setup_kernel (C3/C3b/C10),
// consumed by march_kernel.  Plain words: copied to shared memory per CTA.
struct FrameParams {
    const void* data;          // volume layout base
    int32_t layout, nx, ny, nz;
    int32_t sy, sz;            // strides in layout elements (y, z)
    float supp[3];             // n_a + 1 (support upper bound in padded index space)
    int32_t projection, W, H;
    float inv_dx;
    float B[3], Ex[3], Ey[3], Dg[3];
    float Oe[3], F0[3], fwd[3];
    float Ln[4][3], Lg[4][3], P[4], rgb[4][3];
    uint32_t frame_id;
    int32_t front_ok;          // C9 preconditions hold for this frame
    const uint32_t* occ;       // occupancy bitmask (global), staged to shared memory per CTA
    int32_t occ_shift, occ_nbx, occ_nby, occ_words;   // occ_words: mask + slab boxes (staged)
    int32_t occ_nbz;
    // per-frame helpers for the conservative (estimate-only) computations:
    float invD[3];             // ortho: 1/D_g per axis (0 where D_g = 0)
    float lim[4][3];           // light march exit plane per axis (n+1, 0, or 3e38 if L = 0)
    float ilh[4][3];           // 1 / (L_g * h_l) per axis (1 if L = 0)
    int32_t pair12;            // guide set: light 2 == -light 1 bit-exactly (paired side march)
    // occupied box [alo, ahi) in padded-index positions: every sample outside it is exactly 0
    float alo[3], ahi[3];
    float alim[4][3];          // light march exit plane of the occupied box per axis
    int32_t slab_off;          // word offset of the slab boxes in the staged occupancy region
    int32_t lz0;               // bit l: L_g,l,z == 0 exactly (the march of light l stays in its z slab)
    uint32_t jh;               // C4: the per-frame prefix of the jitter chain, fmix32^3 of (seed, frame)
    int32_t pad2[2];
    // the guide pair's per-occupied-sample constants packed for vector loads (copies of the fields
    // above): (Lg[1], ilh[1][0]), (ilh[1][1], ilh[1][2], 0, 0), (slab_off, occ_nbz, lz0, pair12)
    float4 pk_l1, pk_i1;
    int4 pk_geo;
};
static_assert(sizeof(FrameParams) % 16 == 0, "FrameParams must be 16-B multiple");

// Parameters common to every frame of a call (kernel argument).
// element strides (y, z) of a volume layout, in cells (bricks for BRICK_OCT_F32)
__host__ __device__ inline void layout_strides(int layout, int nx, int ny, int32_t& sy, int32_t& sz) {
    if (layout == NSL_LAYOUT_LINEAR_F32) {            // apron of 1 on each side
        sy = nx + 2;
        sz = (nx + 2) * (ny + 2);
    } else if (layout == NSL_LAYOUT_BRICK_OCT_F32) {  // strides in bricks of 4^3 cells
        sy = (nx + 4) / 4;
        sz = ((nx + 4) / 4) * ((ny + 4) / 4);
    } else if (layout == NSL_LAYOUT_MORTON_OCT_F32) { // strides in tiles of 8^3 cells
        sy = (nx + 8) / 8;
        sz = ((nx + 8) / 8) * ((ny + 8) / 8);
    } else {
        sy = nx + 1;
        sz = (nx + 1) * (ny + 1);
    }
}

// Per (frame, 16x8 tile) of an orthographic march, written by tile_cull_kernel: bits (bit 0: the
// tile's rays miss the occupied box, bit 1: they miss the support box) and [t0, t1], a
// conservative ray-parameter range outside which every sample of every ray of the tile is
// exactly 0 (the union of the tile bundle's hits on the z-slabs' 2-D boxes of occupied blocks).
struct TileCull {
    float t0, t1;
    uint32_t bits, pad;
};

struct MarchConst {
    float h, hl, tau_d, t_min;
    float kappa, alpha, g;
    int32_t Ncap;              // N or 2^24 (unbounded)
    int32_t form, jitter, n_lights, light_mode;
    uint32_t seed_lo, seed_hi;
    int32_t front_identity;
    float axis[3];
    int32_t light_model;       // NSL_LIGHT_MARCH | NSL_LIGHT_TV
    int32_t frame_major;       // march grid order (march.cu): 0 frames fastest, 1 tiles fastest
    int32_t split_k;           // > 0: small FAST guide-set ortho batch -> march_split_kernel with this
                               // bound on the occupied samples of a ray (0: the one-warp-per-tile march)
};

// NEXT-4 transmittance volume: per (frame, lattice slot) constants of the
// light step vector's lattice (V2, fp64 -> fp32) and the sweep window (the occupied box's
// lattice range +-2: lookups at occupied samples never leave it).  Lattice values are float2
// (tau+, tau-) at index (j * Kstr + k) * Astr + i of the slot's block of a group buffer.
struct TvParams {
    float e1[3], e2[3], d[3], dk[3];   // dk = dhat / ell
    float a0, b0, k0, kh;              // lattice offsets (exact small integers), kappa * h_l
    int32_t A, B, K;                   // lattice dims (V2)
    int32_t i_lo, i_hi, j_lo, j_hi, k_lo, k_hi;
    int32_t pad[3];
};
static_assert(sizeof(TvParams) % 16 == 0, "TvParams must be 16-B multiple");
struct TvArgs {                        // march kernel argument (light_model == NSL_LIGHT_TV)
    const TvParams* params;            // [F][slots] (group base)
    const float2* buf;                 // group lattice buffer
    int32_t slots, Astr, Kstr;
    int64_t slot_elems;                // Astr * Bstr * Kstr
};
cudaError_t launch_tv_setup(const FrameParams* fps, int F, int slots, const MarchConst& mc, TvParams* out,
                            cudaStream_t s);
cudaError_t launch_tv_sweep(const FrameParams* fps, const TvParams* tvp, int F, int slots, int Astr, int Bstr,
                            int Kstr, const MarchConst& mc, int layout, float2* buf, cudaStream_t s);

// NEXT-1 six-way bake: per-frame light constants and call constants.
struct BakeFrame {
    float Lg[6][3], Ln[6][3], P[6];
    float lim[6][3], ilh[6][3], alim[6][3];
    int32_t lz0;
    int32_t pad[3];
};
struct BakeConst {
    float hb, hbl, kappa, alpha, g, t_min;
    int32_t spp, Ncap;
    uint32_t seed_lo, seed_hi;
    unsigned long long* counters;   // NULL or [0] += trilinear gathers executed
};

// NEXT-2/3 relight + composite + depth shadow
struct RelightIn {                  // raw per-frame input
    nsl_camera cam;
    nsl_light lights[4];
    nsl_camera shadow_cam[4];
    const float* shadow_map[4];     // device, or NULL (no shadow for that light)
};
// Per-frame constants (fp64 -> fp32 once, by relight_setup_kernel).  Channels ch of a pixel:
// 0 right(+x) 1 top(+y) 2 back(-z) 3 T | 4 left(-x) 5 bottom(-y) 6 front(+z) 7 E (Fig. 2).
struct RelightShadowed {            // a light with a shadow map
    float w[8];                     // R1 weights |c_p| on the selected channels (0 on 3, 7)
    float rgb[3];
    float q[3][4];                  // fi, fj, z = q0 + px q1 + py q2 + D q3 (ortho view), or
    float g[3][3];                  //           = q0 + D (dir . g)            (persp view)
    int32_t Ws, Hs;
    const float* map;
};
struct RelightFrame {
    float M[3][8];                  // unshadowed lights (R1+R2) + composite (bg on ch 3, emis on ch 7)
    float W0[3], Ex[3], Ey[3], F0[3];   // pixel ray (ortho origin / persp direction of pixel (0,0))
    int32_t ns, projection;         // number of shadowed lights
    RelightShadowed sl[4];
};
struct RelightConst {
    int32_t F, W, H, n_lights, any_shadow;
    float bias;
    float bg[3], emis[3];
};
cudaError_t launch_relight(const RelightIn* in, int F, int n_lights, RelightFrame* frames, const RelightConst& rc,
                           const float4* maps, const float* depth, float4* out, cudaStream_t s);

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may start while
// its predecessor in the stream runs, once every CTA of the predecessor has called
// pdl_trigger(); it must call pdl_wait() (full completion + visibility of the predecessor)
// before touching anything the predecessor writes.  Both are no-ops without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();            // NSL_PDL=0 disables the attribute (A/B measurement)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// layouts
constexpr int kLinearF32 = NSL_LAYOUT_LINEAR_F32;
constexpr int kQuadF32 = NSL_LAYOUT_QUAD_F32;
constexpr int kCornerF16 = NSL_LAYOUT_CORNER_F16;
constexpr int kOctF32 = NSL_LAYOUT_OCT_F32;
constexpr int kBrickOctF32 = NSL_LAYOUT_BRICK_OCT_F32;
constexpr int kTex3dF32 = NSL_LAYOUT_TEX3D_F32;
constexpr int kMortonOctF32 = NSL_LAYOUT_MORTON_OCT_F32;

// Launch helpers implemented in the .cu files.
// layout + occupancy + AABB + invalid-voxel count from the raw grid (two launches, no memsets)
cudaError_t launch_volume_build(const float* raw, const VolDesc& v, void* storage, uint32_t* scratch,
                                unsigned long long* invalid, cudaStream_t s);
// sampler microbenchmark (microbench.cu): volume fields of p only
cudaError_t launch_l1_gather(const FrameParams& p, int blocks, int reps, float* sink, cudaStream_t s);
cudaError_t launch_pack_half(const float* rgbt, const float* depth, uint16_t* rgbt_h, uint16_t* depth_h, size_t n,
                             cudaStream_t s);
int l1_gather_threads();
int l1_gather_line();
int l1_gather_max_blocks_per_sm(int layout);
cudaError_t launch_tex_filter(cudaTextureObject_t t, const float* pos, int n, float* out, cudaStream_t s);
int l1_peak_threads();
int l1_peak_patterns();
int l1_peak_max_blocks_per_sm();
cudaError_t launch_l1_peak(const float* buf, const int* lane_off, long long stride, long long span, int blocks,
                           int reps, float* sink, cudaStream_t s);
cudaError_t launch_frame_setup(const FrameIn* in, const nsl_light* lights, int F, const MarchConst& mc,
                               FrameParams* out, cudaStream_t s);
// mode: 0 fast (timed path), 1 debug (canonical counters, no shortcuts), 2 counted fast path.
// cull: march_cull_bytes(F, W, H) bytes of device workspace (orthographic views: a TileCull per tile).
// tv: NULL (light_model 0) or the group's transmittance-volume arguments.
cudaError_t launch_march(const FrameParams* fp, const MarchConst& mc, int F, int W, int H, int projection,
                         int layout, float4* rgbt, float* depth, uint32_t* debug, unsigned long long* counters,
                         TileCull* cull, const TvArgs* tv, cudaStream_t s);
size_t march_cull_bytes(int F, int W, int H);
int march_tile_w();
int march_split_max_k();
int march_tile_h();
cudaError_t launch_bake_setup(const FrameIn* in, const FrameParams* fps, int F, float hbl, float g, BakeFrame* out,
                              cudaStream_t s);
cudaError_t launch_bake(const FrameParams* fp, const BakeFrame* bf, const BakeConst& bc, int F, int W, int H,
                        int projection, int layout, float4* out, cudaStream_t s);
cudaError_t launch_jitter_debug(const MarchConst& mc, uint32_t frame_id, int n, uint32_t* hash, float* delta,
                                cudaStream_t s);

size_t layout_elems(int layout, int nx, int ny, int nz);
size_t layout_elem_bytes(int layout);

}  // namespace nsl
