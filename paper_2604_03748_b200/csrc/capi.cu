// capi.cu — the C ABI of include/nsl.h: argument validation, volume handles,
// per-call frame tables, kernel dispatch.  Host code only; every step of the
// guiding-map path runs in the kernels of volume.cu / setup.cu / march.cu.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "nsl_internal.cuh"

using namespace nsl;

struct nsl_volume {
    nsl_grid_desc g;
    int32_t layout;
    void* data;                       // caller-owned storage: layout body | occupancy mask | tail
    unsigned long long* invalid;      // counter in the storage tail
    uint32_t* occ;                    // occupancy bitmask inside the storage
    nsl::OccGeom og;
    int32_t* aabb;                    // occupied block bounds in the storage tail
    // TEX3D only: the library-owned body (QUAD float4 texels) and its texture / surface objects
    cudaArray_t arr = nullptr;
    cudaTextureObject_t tex = 0;
    cudaSurfaceObject_t surf = 0;
    ~nsl_volume() {
        if (tex) cudaDestroyTextureObject(tex);
        if (surf) cudaDestroySurfaceObject(surf);
        if (arr) cudaFreeArray(arr);
    }
};

namespace {

thread_local std::string g_err;

nsl_status fail(nsl_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

nsl_status cuda_fail(cudaError_t e, const char* what) {
    return fail(e == cudaErrorMemoryAllocation ? NSL_ERR_OUT_OF_MEMORY : NSL_ERR_CUDA, "%s: %s", what,
                cudaGetErrorString(e));
}

#define NSL_CUDA(call, what)                       \
    do {                                           \
        cudaError_t e_ = (call);                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

bool finite3(const float v[3]) { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); }
double norm3(const float v[3]) {
    return std::sqrt((double)v[0] * v[0] + (double)v[1] * v[1] + (double)v[2] * v[2]);
}

constexpr size_t kTail = 256;  // counter area after the layout (keeps 16-B alignment)

size_t body_bytes(const nsl_grid_desc* g, int layout) {
    return layout_elems(layout, g->nx, g->ny, g->nz) * layout_elem_bytes(layout);
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// storage = [layout body | occupancy region | build scratch | tail counter], each 256-B aligned
size_t mask_offset(const nsl_grid_desc* g, int layout) { return align_up(body_bytes(g, layout), 256); }
size_t scratch_offset(const nsl_grid_desc* g, int layout) {
    return mask_offset(g, layout) + align_up((size_t)occ_geom(g->nx, g->ny, g->nz).words_total * 4, 256);
}
size_t tail_offset(const nsl_grid_desc* g, int layout) {
    return scratch_offset(g, layout) + align_up((size_t)occ_geom(g->nx, g->ny, g->nz).scratch_words * 4, 256);
}

nsl_status check_grid(const nsl_grid_desc* g) {
    if (!g) return fail(NSL_ERR_INVALID_ARG, "grid descriptor is NULL");
    if (g->nx < 1 || g->ny < 1 || g->nz < 1) return fail(NSL_ERR_INVALID_ARG, "grid dims must be >= 1");
    if (!(g->voxel_width > 0.0f) || !std::isfinite(g->voxel_width))
        return fail(NSL_ERR_INVALID_ARG, "voxel_width must be finite and > 0");
    if (!finite3(g->origin)) return fail(NSL_ERR_INVALID_ARG, "grid origin must be finite");
    double cells = (double)(g->nx + 2) * (g->ny + 2) * (g->nz + 2);
    if (cells >= 2147483647.0) return fail(NSL_ERR_UNSUPPORTED, "grid too large for 32-bit indexing");
    return NSL_OK;
}

// NSL_LAYOUT_AUTO (the default): the layout chosen from the grid size by measurement (DESIGN.md §6,
// profiles/r2_per_config): BRICK_OCT_F32 once the OCT body exceeds 2 GiB (C5's 512^3 static
// volume: march -6.7 % over the 1024-frame batch), OCT_F32 below (C2 128^3: BRICK +3 %; C3 256^3:
// equal, and BRICK's build costs 2x).  Animated volumes (a build per frame) resolve to OCT_F32.
int resolve_layout(const nsl_grid_desc* g, int layout, bool animated = false) {
    if (layout != NSL_LAYOUT_AUTO || !g) return layout;
    if (animated) return kOctF32;
    const double body = (double)(g->nx + 1) * (g->ny + 1) * (g->nz + 1) * 32.0;
    return body > 2147483648.0 ? kBrickOctF32 : kOctF32;
}

nsl_status check_layout(int layout) {
    if (layout != kLinearF32 && layout != kQuadF32 && layout != kCornerF16 && layout != kOctF32 &&
        layout != kBrickOctF32 && layout != kTex3dF32 && layout != kMortonOctF32)
        return fail(NSL_ERR_INVALID_ARG, "unknown layout %d", layout);
    return NSL_OK;
}

nsl_status check_camera(const nsl_camera* c, int idx) {
    if (c->projection != 0 && c->projection != 1) return fail(NSL_ERR_INVALID_ARG, "camera[%d]: bad projection", idx);
    if (c->width < 1 || c->height < 1) return fail(NSL_ERR_INVALID_ARG, "camera[%d]: width/height must be >= 1", idx);
    if ((double)c->width * c->height >= 2147483647.0)
        return fail(NSL_ERR_UNSUPPORTED, "camera[%d]: image too large", idx);
    if (!finite3(c->position) || !finite3(c->forward) || !finite3(c->up))
        return fail(NSL_ERR_INVALID_ARG, "camera[%d]: non-finite vector", idx);
    if (!(c->extent > 0.0f) || !std::isfinite(c->extent))
        return fail(NSL_ERR_INVALID_ARG, "camera[%d]: extent must be finite and > 0", idx);
    double nf = norm3(c->forward);
    if (std::fabs(nf - 1.0) > 1e-3) return fail(NSL_ERR_INVALID_ARG, "camera[%d]: |forward| = %g is not unit", idx, nf);
    double nu = norm3(c->up);
    if (!(nu > 0.0)) return fail(NSL_ERR_INVALID_ARG, "camera[%d]: up is zero", idx);
    double cx = (double)c->forward[1] * c->up[2] - (double)c->forward[2] * c->up[1];
    double cy = (double)c->forward[2] * c->up[0] - (double)c->forward[0] * c->up[2];
    double cz = (double)c->forward[0] * c->up[1] - (double)c->forward[1] * c->up[0];
    if (std::sqrt(cx * cx + cy * cy + cz * cz) < 1e-4 * nf * nu)
        return fail(NSL_ERR_INVALID_ARG, "camera[%d]: up is parallel to forward", idx);
    return NSL_OK;
}

nsl_status check_lights(const nsl_light* l, int n, int mode, int idx) {
    for (int i = 0; i < n; ++i) {
        if (!finite3(l[i].rgb) || l[i].rgb[0] < 0 || l[i].rgb[1] < 0 || l[i].rgb[2] < 0)
            return fail(NSL_ERR_INVALID_ARG, "light[%d][%d]: rgb must be finite and >= 0", idx, i);
        if (mode == NSL_LIGHTS_EXPLICIT) {
            if (!finite3(l[i].to_light)) return fail(NSL_ERR_INVALID_ARG, "light[%d][%d]: non-finite direction", idx, i);
            double nl = norm3(l[i].to_light);
            if (std::fabs(nl - 1.0) > 1e-3)
                return fail(NSL_ERR_INVALID_ARG, "light[%d][%d]: |to_light| = %g is not unit", idx, i, nl);
        }
    }
    return NSL_OK;
}

nsl_status check_common(const nsl_light* lights, int n_lights, int light_mode, const nsl_medium* med,
                        const nsl_march* m) {
    if (!lights) return fail(NSL_ERR_INVALID_ARG, "lights is NULL");
    if (!med || !m) return fail(NSL_ERR_INVALID_ARG, "medium/march is NULL");
    if (light_mode != NSL_LIGHTS_EXPLICIT && light_mode != NSL_LIGHTS_GUIDE)
        return fail(NSL_ERR_INVALID_ARG, "bad light_mode %d", light_mode);
    if (n_lights < 1 || n_lights > 4) return fail(NSL_ERR_INVALID_ARG, "n_lights must be in [1,4]");
    if (light_mode == NSL_LIGHTS_GUIDE && n_lights > 3) return fail(NSL_ERR_INVALID_ARG, "guide set has at most 3 lights");
    if (!(med->extinction >= 0.0f) || !std::isfinite(med->extinction))
        return fail(NSL_ERR_INVALID_ARG, "extinction must be finite and >= 0");
    if (!(med->albedo >= 0.0f && med->albedo <= 1.0f)) return fail(NSL_ERR_INVALID_ARG, "albedo must be in [0,1]");
    if (!(med->hg_g > -1.0f && med->hg_g < 1.0f)) return fail(NSL_ERR_INVALID_ARG, "hg_g must be in (-1,1)");
    if (!(m->step > 0.0f) || !std::isfinite(m->step)) return fail(NSL_ERR_INVALID_ARG, "step must be finite and > 0");
    if (!(m->light_step >= 0.0f) || !std::isfinite(m->light_step))
        return fail(NSL_ERR_INVALID_ARG, "light_step must be finite and >= 0");
    if (m->max_steps < 0 || m->max_steps > (1 << 24)) return fail(NSL_ERR_INVALID_ARG, "max_steps out of range");
    if (!(m->depth_tau >= 0.0f) || !std::isfinite(m->depth_tau))
        return fail(NSL_ERR_INVALID_ARG, "depth_tau must be finite and >= 0");
    if (!(m->t_min >= 0.0f && m->t_min < 1.0f)) return fail(NSL_ERR_INVALID_ARG, "t_min must be in [0,1)");
    if (m->opacity_form < 0 || m->opacity_form > 2) return fail(NSL_ERR_INVALID_ARG, "bad opacity_form");
    if (m->jitter != 0 && m->jitter != 1) return fail(NSL_ERR_INVALID_ARG, "jitter must be 0 or 1");
    if (!finite3(m->guide_axis)) return fail(NSL_ERR_INVALID_ARG, "guide_axis must be finite");
    if (m->light_model != NSL_LIGHT_MARCH && m->light_model != NSL_LIGHT_TV)
        return fail(NSL_ERR_INVALID_ARG, "bad light_model %d", m->light_model);
    return NSL_OK;
}

MarchConst make_const(int n_lights, int light_mode, const nsl_medium* med, const nsl_march* m) {
    MarchConst mc;
    mc.h = m->step;
    mc.hl = m->light_step > 0.0f ? m->light_step : m->step;
    mc.tau_d = m->depth_tau;
    mc.t_min = m->t_min;
    mc.kappa = med->extinction;
    mc.alpha = med->albedo;
    mc.g = med->hg_g;
    mc.Ncap = m->max_steps > 0 ? m->max_steps : (1 << 24);
    mc.form = m->opacity_form;
    mc.jitter = m->jitter;
    mc.n_lights = n_lights;
    mc.light_mode = light_mode;
    mc.seed_lo = (uint32_t)(m->seed & 0xffffffffu);
    mc.seed_hi = (uint32_t)(m->seed >> 32);
    mc.front_identity = m->front_identity ? 1 : 0;
    mc.axis[0] = m->guide_axis[0];
    mc.axis[1] = m->guide_axis[1];
    mc.axis[2] = m->guide_axis[2];
    mc.light_model = m->light_model;
    mc.frame_major = 0;
    mc.split_k = 0;
    return mc;
}

VolDesc desc_of(const nsl_volume* v) {
    VolDesc d;
    d.data = v->data;
    d.nx = v->g.nx;
    d.ny = v->g.ny;
    d.nz = v->g.nz;
    d.layout = v->layout;
    d.origin[0] = v->g.origin[0];
    d.origin[1] = v->g.origin[1];
    d.origin[2] = v->g.origin[2];
    d.dx = v->g.voxel_width;
    d.occ = v->occ;
    d.og = v->og;
    d.aabb = v->aabb;
    if (v->layout == kTex3dF32) d.data = reinterpret_cast<const void*>((uintptr_t)v->tex);   // kernels: the texture
    d.surf = v->surf;
    return d;
}

// Stream-ordered allocations of the library (frame tables, host-API staging, TV lattices) come
// from a library-private pool per device, never the device's default pool that torch and other
// libraries share.  Up to NSL_POOL_RETAIN_MB (default 4096, ~2 % of the B200's 180 GB) of it
// is retained across
// synchronisations, so per-call tables and the host API's staging are recycled instead of
// re-mapped each call; anything above is released at the next synchronisation (e.g. the
// transient TV lattices of up to NSL_TV_BUDGET_MB).
cudaError_t pool_malloc_v(void** p, size_t bytes, cudaStream_t s) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!pools[dev]) {
            cudaMemPoolProps props;
            memset(&props, 0, sizeof props);
            props.allocType = cudaMemAllocationTypePinned;
            props.handleTypes = cudaMemHandleTypeNone;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            cudaMemPool_t np = nullptr;
            e = cudaMemPoolCreate(&np, &props);
            if (e != cudaSuccess) return e;
            // 4 GiB: the host API's transient buffers for C3-size batches (1.3 GB of fp32 maps,
            // 1.9 GB with the fp16 staging) stay mapped between calls; at 1 GiB they were re-mapped
            // every call (C3 e2e varied 10x between runs)
            double mb = 4096.0;
            if (const char* env = getenv("NSL_POOL_RETAIN_MB")) mb = atof(env);
            uint64_t thr = mb <= 0.0 ? 0 : (uint64_t)(mb * 1048576.0);
            cudaMemPoolSetAttribute(np, cudaMemPoolAttrReleaseThreshold, &thr);
            pools[dev] = np;
        }
        pool = pools[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}
template <class T>
cudaError_t pool_malloc(T** p, size_t bytes, cudaStream_t s) {
    return pool_malloc_v(reinterpret_cast<void**>(p), bytes, s);
}

// Frame tables: FrameIn[F] | lights[F*nl] | FrameParams[F] in one stream-ordered allocation.
struct Workspace {
    void* base = nullptr;
    FrameIn* in = nullptr;
    nsl_light* lights = nullptr;
    FrameParams* params = nullptr;
    TileCull* cull = nullptr;          // march_cull_bytes workspace (march calls only)
};

// The frame tables (FrameIn, lights) uploaded into a fresh stream-ordered workspace, plus the
// march's tile cull flags when `march`.
nsl_status upload_frames(const std::vector<FrameIn>& frames, const nsl_light* lights, int n_lights, bool march,
                         cudaStream_t s, Workspace& ws) {
    const int F = (int)frames.size();
    const size_t b_in = align_up(sizeof(FrameIn) * F, 256);
    const size_t b_l = align_up(sizeof(nsl_light) * (size_t)F * n_lights, 256);
    const size_t b_p = align_up(sizeof(FrameParams) * F, 256);
    const size_t b_c = march ? march_cull_bytes(F, frames[0].cam.width, frames[0].cam.height) : 0;
    NSL_CUDA(pool_malloc(&ws.base, b_in + b_l + b_p + b_c, s), "cudaMallocAsync(frame tables)");
    ws.in = reinterpret_cast<FrameIn*>(ws.base);
    ws.lights = reinterpret_cast<nsl_light*>(static_cast<char*>(ws.base) + b_in);
    ws.params = reinterpret_cast<FrameParams*>(static_cast<char*>(ws.base) + b_in + b_l);
    ws.cull = b_c ? reinterpret_cast<TileCull*>(static_cast<char*>(ws.base) + b_in + b_l + b_p) : nullptr;
    std::vector<char> host(b_in + b_l);
    memcpy(host.data(), frames.data(), sizeof(FrameIn) * F);
    memcpy(host.data() + b_in, lights, sizeof(nsl_light) * (size_t)F * n_lights);
    NSL_CUDA(cudaMemcpyAsync(ws.base, host.data(), host.size(), cudaMemcpyHostToDevice, s), "frame table upload");
    return NSL_OK;
}

nsl_status build_frames(const std::vector<FrameIn>& frames, const nsl_light* lights, int n_lights,
                        const MarchConst& mc, bool march, cudaStream_t s, Workspace& ws) {
    if (nsl_status st = upload_frames(frames, lights, n_lights, march, s, ws)) return st;
    NSL_CUDA(launch_frame_setup(ws.in, ws.lights, (int)frames.size(), mc, ws.params, s), "frame_setup_kernel launch");
    return NSL_OK;
}

}  // namespace

extern "C" {

const char* nsl_last_error(void) { return g_err.c_str(); }
const char* nsl_version(void) { return "nsl-b200 0.1 (sm_100a)"; }

int32_t nsl_layout_resolve(const nsl_grid_desc* g, int32_t layout) {
    if (check_grid(g) != NSL_OK) return -1;
    return resolve_layout(g, layout);
}

int32_t nsl_volume_build_launches(const nsl_grid_desc* g, int32_t layout) {
    if (check_grid(g) != NSL_OK) return -1;
    layout = resolve_layout(g, layout);
    if (check_layout(layout) != NSL_OK) return -1;
    return staged_oct_build(layout, occ_geom(g->nx, g->ny, g->nz)) ? 3 : 2;
}

size_t nsl_volume_bytes(const nsl_grid_desc* g, int32_t layout) {
    layout = resolve_layout(g, layout);
    if (check_grid(g) != NSL_OK || check_layout(layout) != NSL_OK) return 0;
    return tail_offset(g, layout) + kTail;
}

static nsl_status volume_upload_impl(const nsl_grid_desc* g, const float* density, int32_t density_on_device,
                                     int32_t layout, void* device_storage, size_t storage_bytes, nsl_stream stream,
                                     nsl_volume** out, bool validate_host);

// Host-only part of an upload: argument checks and the handle (no device work).
static nsl_status volume_handle(const nsl_grid_desc* g, int32_t layout, void* device_storage, size_t storage_bytes,
                                nsl_volume** out) {
    layout = resolve_layout(g, layout);
    if (nsl_status st = check_grid(g)) return st;
    if (nsl_status st = check_layout(layout)) return st;
    if (!device_storage) return fail(NSL_ERR_INVALID_ARG, "NULL storage");
    const int align = layout == kOctF32 || layout == kBrickOctF32 || layout == kMortonOctF32 ? 32 : 16;
    if (reinterpret_cast<uintptr_t>(device_storage) % align)
        return fail(NSL_ERR_INVALID_ARG, "storage must be %d-B aligned", align);
    const size_t need = nsl_volume_bytes(g, layout);
    if (storage_bytes < need) return fail(NSL_ERR_INVALID_ARG, "storage_bytes %zu < required %zu", storage_bytes, need);
    nsl_volume* v = new nsl_volume;
    v->g = *g;
    v->layout = layout;
    v->data = device_storage;
    v->invalid = reinterpret_cast<unsigned long long*>(static_cast<char*>(device_storage) + tail_offset(g, layout));
    v->occ = reinterpret_cast<uint32_t*>(static_cast<char*>(device_storage) + mask_offset(g, layout));
    v->og = occ_geom(g->nx, g->ny, g->nz);
    v->aabb = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(v->invalid) + 16);
    if (layout == kTex3dF32) {
        // the body: (nx+1) x (ny+1) x (nz+2) QUAD float4 texels in a 3-D cudaArray (block-linear),
        // written by the build through a surface, read by the march through a point-sampled,
        // unnormalised texture (clamp addressing: every fetch is in range by construction)
        const cudaChannelFormatDesc cd = cudaCreateChannelDesc<float4>();
        cudaError_t e = cudaMalloc3DArray(&v->arr, &cd, make_cudaExtent(g->nx + 1, g->ny + 1, g->nz + 2),
                                          cudaArraySurfaceLoadStore);
        cudaResourceDesc rd;
        memset(&rd, 0, sizeof rd);
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = v->arr;
        cudaTextureDesc td;
        memset(&td, 0, sizeof td);
        td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModePoint;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        if (e == cudaSuccess) e = cudaCreateTextureObject(&v->tex, &rd, &td, nullptr);
        if (e == cudaSuccess) e = cudaCreateSurfaceObject(&v->surf, &rd);
        if (e != cudaSuccess) {
            delete v;
            return cuda_fail(e, "TEX3D array / texture");
        }
    }
    *out = v;
    return NSL_OK;
}

// Device part: the layout + occupancy build of a device-resident raw grid into v's storage.
static cudaError_t enqueue_build(const nsl_volume* v, const float* raw, cudaStream_t s) {
    return launch_volume_build(
        raw, desc_of(v), v->data,
        reinterpret_cast<uint32_t*>(static_cast<char*>(v->data) + scratch_offset(&v->g, v->layout)), v->invalid, s);
}

nsl_status nsl_volume_upload(const nsl_grid_desc* g, const float* density, int32_t density_on_device, int32_t layout,
                             void* device_storage, size_t storage_bytes, nsl_stream stream, nsl_volume** out) {
    return volume_upload_impl(g, density, density_on_device, layout, device_storage, storage_bytes, stream, out, true);
}

// validate_host = false: host values are checked on the device only (the build kernel's
// invalid-voxel count); the caller must read it (nsl_guiding_map_host does, after its sync).
static nsl_status volume_upload_impl(const nsl_grid_desc* g, const float* density, int32_t density_on_device,
                                     int32_t layout, void* device_storage, size_t storage_bytes, nsl_stream stream,
                                     nsl_volume** out, bool validate_host) {
    g_err.clear();
    if (!density || !out) return fail(NSL_ERR_INVALID_ARG, "NULL density/out");
    nsl_volume* v = nullptr;
    if (nsl_status st = volume_handle(g, layout, device_storage, storage_bytes, &v)) return st;
    const size_t n = (size_t)g->nx * g->ny * g->nz;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto bail = [&](nsl_status st) { delete v; return st; };
    if (!density_on_device && validate_host) {
        for (size_t i = 0; i < n; ++i)
            if (!(density[i] >= 0.0f) || !std::isfinite(density[i]))
                return bail(fail(NSL_ERR_INVALID_ARG, "density[%zu] = %g is not finite and >= 0", i,
                                 (double)density[i]));
    }
    cudaError_t e = cudaSuccess;
    const float* raw = density;
    void* staging = nullptr;
    // nsl.h: host density may be reused as soon as nsl_volume_upload returns.  A copy from
    // pinned memory is still in flight after cudaMemcpyAsync (pageable sources are staged
    // synchronously by the driver), so the call waits for the copy -- not for the build, which
    // stays asynchronous.  (The host API, validate_host = false, owns that lifetime itself.)
    cudaEvent_t copied = nullptr;
    auto drop = [&](nsl_status st) { if (copied) cudaEventDestroy(copied); return bail(st); };
    if (!density_on_device) {
        e = pool_malloc(&staging, n * sizeof(float), s);
        if (e != cudaSuccess) return bail(cuda_fail(e, "cudaMallocAsync(staging)"));
        e = cudaMemcpyAsync(staging, density, n * sizeof(float), cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return bail(cuda_fail(e, "density upload"));
        if (validate_host) {
            e = cudaEventCreateWithFlags(&copied, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventRecord(copied, s);
            if (e != cudaSuccess) return drop(cuda_fail(e, "density upload event"));
        }
        raw = static_cast<const float*>(staging);
    }
    e = enqueue_build(v, raw, s);
    if (e != cudaSuccess) return drop(cuda_fail(e, "volume build launch"));
    if (staging) {
        e = cudaFreeAsync(staging, s);
        if (e != cudaSuccess) return drop(cuda_fail(e, "cudaFreeAsync(staging)"));
    }
    if (copied) {
        e = cudaEventSynchronize(copied);
        cudaEventDestroy(copied);
        copied = nullptr;
        if (e != cudaSuccess) return bail(cuda_fail(e, "density upload wait"));
    }
    *out = v;
    return NSL_OK;
}

nsl_status nsl_volume_check(const nsl_volume* v, nsl_stream stream, uint64_t* n_invalid) {
    g_err.clear();
    if (!v || !n_invalid) return fail(NSL_ERR_INVALID_ARG, "NULL volume/out");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    unsigned long long h = 0;
    NSL_CUDA(cudaMemcpyAsync(&h, v->invalid, sizeof h, cudaMemcpyDeviceToHost, s), "invalid counter read");
    NSL_CUDA(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    *n_invalid = h;
    return NSL_OK;
}

nsl_status nsl_volume_release(nsl_volume* v) {
    delete v;
    return NSL_OK;
}

nsl_status nsl_volume_rebuild(nsl_volume* v, const float* density, int32_t density_on_device, nsl_stream stream) {
    g_err.clear();
    if (!v || !density) return fail(NSL_ERR_INVALID_ARG, "NULL volume/density");
    const size_t n = (size_t)v->g.nx * v->g.ny * v->g.nz;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (density_on_device) {
        NSL_CUDA(enqueue_build(v, density, s), "volume build launch");
        return NSL_OK;
    }
    for (size_t i = 0; i < n; ++i)
        if (!(density[i] >= 0.0f) || !std::isfinite(density[i]))
            return fail(NSL_ERR_INVALID_ARG, "density[%zu] = %g is not finite and >= 0", i, (double)density[i]);
    void* staging = nullptr;
    NSL_CUDA(pool_malloc(&staging, n * sizeof(float), s), "cudaMallocAsync(staging)");
    cudaError_t e = cudaMemcpyAsync(staging, density, n * sizeof(float), cudaMemcpyHostToDevice, s);
    cudaEvent_t copied = nullptr;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&copied, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(copied, s);
    if (e == cudaSuccess) e = enqueue_build(v, static_cast<const float*>(staging), s);
    cudaError_t e2 = cudaFreeAsync(staging, s);
    if (e == cudaSuccess && copied) e = cudaEventSynchronize(copied);   // host buffer reusable on return
    if (copied) cudaEventDestroy(copied);
    if (e != cudaSuccess) return cuda_fail(e, "volume rebuild");
    if (e2 != cudaSuccess) return cuda_fail(e2, "cudaFreeAsync(staging)");
    return NSL_OK;
}

// March grid order: tiles fastest (the CTAs in flight cover one frame and share
// its volume) when the frames view different volumes; frames fastest when they share one (the
// CTAs in flight then cover the same tile of consecutive frames, whose nearby cameras read
// nearly the same cells, and the launch tail is made of cheap border tiles).  Measured: C4
// (a volume per frame) march 3.23 -> 1.55 ms; C2 / C3 / C5 (one volume) +3 % / +10 % / +38 %
// with tiles fastest.  NSL_FRAME_MAJOR=0/1 forces either.
static int32_t march_frame_major(const std::vector<FrameIn>& frames) {
    if (const char* e = getenv("NSL_FRAME_MAJOR")) return atoi(e) != 0;
    for (const FrameIn& f : frames)
        if (f.vol.data != frames[0].vol.data) return 1;
    return 0;
}

// Validated, marshalled form of a batch call (host side only).
struct Prepared {
    std::vector<FrameIn> frames;
    MarchConst mc;
    int F = 0, W = 0, H = 0, proj = 0, layout = 0, n_lights = 0;
    // NEXT-4 transmittance volume (light_model == NSL_LIGHT_TV): lattice slots per frame, host
    // bounds of the lattice dims (strides), frames per group under the memory budget
    int tv_slots = 0, tv_Astr = 0, tv_Bstr = 0, tv_Kstr = 0, tv_group = 0;
    size_t tv_params_bytes() const { return sizeof(TvParams) * (size_t)F * tv_slots; }
    size_t tv_slot_elems() const { return (size_t)tv_Astr * tv_Bstr * tv_Kstr; }
    size_t tv_buf_bytes() const { return sizeof(float2) * tv_slot_elems() * tv_slots * (size_t)tv_group; }
};

// Split march (march.cu march_split_kernel) for small FAST guide-set orthographic batches, whose
// one-warp-per-tile grid would leave most SMs idle (at most a third of a wave of warps): returns the
// bound K on the occupied samples of a ray -- at most the in-support steps, floor(support
// diagonal / step) + 1 in index units, and at most max_steps -- or 0 (no split: too many warps,
// another light set or model, perspective, the texture layout, or K above the shared-memory
// budget).  The split kernel's maps are bitwise those of march_kernel.  NSL_SPLIT=0/1 forces it
// off / on (when eligible).
static int32_t march_split_k(const Prepared& P) {
    const char* e = getenv("NSL_SPLIT");
    if (e && e[0] == '0') return 0;
    if (P.proj != 0 || P.layout == kTex3dF32 || P.mc.light_model != NSL_LIGHT_MARCH ||
        P.mc.light_mode != NSL_LIGHTS_GUIDE || P.n_lights != 3)
        return 0;
    const long long warps = (long long)P.F * ((P.W + 7) / 8) * ((P.H + 3) / 4);
    // measured (profiles/r2_ab6): C1 (512 warps) step 0.043 -> 0.033 ms; the paper's 512^2 x 400^3
    // frame (8192 warps, over one wave) +4 % (the split's shared memory halves the resident warps)
    const long long third_wave = 148LL * 16;
    if (!(e && e[0] == '1') && warps > third_wave) return 0;
    double kmax = 0.0;
    for (const FrameIn& f : P.frames) {
        const double d = std::sqrt((f.vol.nx + 1.0) * (f.vol.nx + 1.0) + (f.vol.ny + 1.0) * (f.vol.ny + 1.0) +
                                   (f.vol.nz + 1.0) * (f.vol.nz + 1.0));
        const double k = std::floor(d * (double)f.vol.dx / (double)P.mc.h * (1.0 + 1e-6)) + 2.0;
        kmax = k > kmax ? k : kmax;
    }
    if (kmax > (double)P.mc.Ncap) kmax = (double)P.mc.Ncap;
    if (kmax < 1.0 || kmax > (double)march_split_max_k()) return 0;
    return (int32_t)kmax;
}

// Host bounds of the V2 lattice dims: the projection of the support box on
// any unit vector is at most its diagonal, so A, B <= diag + 5 and K <= diag / ell + 5 with
// ell = h_l / voxel_width (unit lights); +6 (and 1e-5 on ell) keeps every device value below.
static void tv_geometry(const nsl_volume* const* vols, int n_vols, Prepared& P) {
    P.tv_slots = 0;
    if (P.mc.light_model != NSL_LIGHT_TV) return;
    P.tv_slots = P.mc.light_mode == NSL_LIGHTS_GUIDE ? (P.n_lights > 1 ? 1 : 0) : P.n_lights;
    if (!P.tv_slots) return;
    double diag = 0.0, kext = 0.0;
    for (int i = 0; i < n_vols; ++i) {
        const nsl_grid_desc& g = vols[i]->g;
        const double d = std::sqrt((g.nx + 1.0) * (g.nx + 1.0) + (g.ny + 1.0) * (g.ny + 1.0) + (g.nz + 1.0) * (g.nz + 1.0));
        diag = d > diag ? d : diag;
        const double k = d / ((double)P.mc.hl / (double)g.voxel_width * (1.0 - 1e-5));
        kext = k > kext ? k : kext;
    }
    P.tv_Astr = P.tv_Bstr = (int)std::ceil(diag) + 6;
    P.tv_Kstr = (int)std::ceil(kext) + 6;
    double budget_mb = 4096.0;   // measured: 1024 -> 4096 MB: C3 TV 2.95 -> 2.87, C5 TV 2.37 -> 2.09 ms
    if (const char* e = getenv("NSL_TV_BUDGET_MB")) budget_mb = atof(e);
    const double per_frame = (double)sizeof(float2) * P.tv_slot_elems() * P.tv_slots;
    const double g = std::floor(budget_mb * 1048576.0 / per_frame);
    P.tv_group = g < 1.0 ? 1 : (g > P.F ? P.F : (int)g);
    // tv_sweep_kernel's grid.y is group * slots (<= 65535)
    if ((long long)P.tv_group * P.tv_slots > 65535) P.tv_group = 65535 / P.tv_slots;
}

// The march of a prepared batch: one launch, or (light_model TV) the lattice setup, then per
// frame group the sweep and the march of that group.  tvp/tvbuf: P.tv_params_bytes() and
// P.tv_buf_bytes() of device workspace (unused otherwise).
static cudaError_t run_march(const Prepared& P, const FrameParams* params, TileCull* cull,
                             TvParams* tvp, float2* tvbuf, float* out_rgbt, float* out_depth, uint32_t* out_debug,
                             unsigned long long* counters, cudaStream_t s) {
    float4* rgbt = reinterpret_cast<float4*>(out_rgbt);
    if (!P.tv_slots)
        return launch_march(params, P.mc, P.F, P.W, P.H, P.proj, P.layout, rgbt, out_depth, out_debug, counters,
                            cull, nullptr, s);
    cudaError_t e = launch_tv_setup(params, P.F, P.tv_slots, P.mc, tvp, s);
    const size_t npf = (size_t)P.W * P.H;
    const size_t tiles = march_cull_bytes(1, P.W, P.H) / sizeof(TileCull);
    for (int g0 = 0; e == cudaSuccess && g0 < P.F; g0 += P.tv_group) {
        const int n = P.F - g0 < P.tv_group ? P.F - g0 : P.tv_group;
        const TvParams* gp = tvp + (size_t)g0 * P.tv_slots;
        e = launch_tv_sweep(params + g0, gp, n, P.tv_slots, P.tv_Astr, P.tv_Bstr, P.tv_Kstr, P.mc, P.layout, tvbuf, s);
        if (e != cudaSuccess) break;
        const TvArgs ta{gp, tvbuf, P.tv_slots, P.tv_Astr, P.tv_Kstr, (int64_t)P.tv_slot_elems()};
        e = launch_march(params + g0, P.mc, n, P.W, P.H, P.proj, P.layout, rgbt + (size_t)g0 * npf,
                         out_depth + (size_t)g0 * npf, out_debug ? out_debug + (size_t)g0 * npf * 6 : nullptr, counters,
                         cull ? cull + (size_t)g0 * tiles : nullptr, &ta, s);
    }
    return e;
}

static nsl_status prepare(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                          const nsl_camera* cams, const nsl_light* lights, int32_t n_lights, int32_t light_mode,
                          const nsl_medium* med, const nsl_march* m, const uint32_t* frame_ids, int32_t F,
                          Prepared& P) {
    if (F < 1 || F > 65535) return fail(NSL_ERR_INVALID_ARG, "F must be in [1, 65535]");
    if (!vols || n_vols < 1 || !frame_vol || !cams || !frame_ids)
        return fail(NSL_ERR_INVALID_ARG, "NULL vols/frame_vol/cams/frame_ids");
    if (nsl_status st = check_common(lights, n_lights, light_mode, med, m)) return st;
    for (int i = 0; i < n_vols; ++i)
        if (!vols[i]) return fail(NSL_ERR_INVALID_ARG, "vols[%d] is NULL", i);
    P.layout = vols[0]->layout;
    for (int i = 0; i < n_vols; ++i)
        if (vols[i]->layout != P.layout) return fail(NSL_ERR_UNSUPPORTED, "all volumes of a batch must share a layout");
    P.W = cams[0].width;
    P.H = cams[0].height;
    if ((long)((P.W + march_tile_w() - 1) / march_tile_w()) * ((P.H + march_tile_h() - 1) / march_tile_h()) > 65535)
        return fail(NSL_ERR_UNSUPPORTED, "image too large: more than 65535 march tiles (16x%d pixels) per frame",
                    march_tile_h());
    P.proj = cams[0].projection;
    P.F = F;
    P.n_lights = n_lights;
    P.frames.assign((size_t)F, FrameIn{});
    for (int f = 0; f < F; ++f) {
        if (nsl_status st = check_camera(&cams[f], f)) return st;
        if (cams[f].width != P.W || cams[f].height != P.H)
            return fail(NSL_ERR_INVALID_ARG, "camera[%d]: size differs", f);
        if (cams[f].projection != P.proj) return fail(NSL_ERR_UNSUPPORTED, "camera[%d]: mixed projections", f);
        if (frame_vol[f] < 0 || frame_vol[f] >= n_vols) return fail(NSL_ERR_INVALID_ARG, "frame_vol[%d] out of range", f);
        if (nsl_status st = check_lights(lights + (size_t)f * n_lights, n_lights, light_mode, f)) return st;
        FrameIn& fi = P.frames[f];
        memset(&fi, 0, sizeof fi);
        fi.cam = cams[f];
        fi.vol = desc_of(vols[frame_vol[f]]);
        fi.frame_id = frame_ids[f];
    }
    P.mc = make_const(n_lights, light_mode, med, m);
    P.mc.frame_major = march_frame_major(P.frames);
    P.mc.split_k = march_split_k(P);
    tv_geometry(vols, n_vols, P);
    return NSL_OK;
}

static nsl_status check_outputs(const float* out_rgbt, const float* out_depth) {
    if (!out_rgbt || !out_depth) return fail(NSL_ERR_INVALID_ARG, "NULL output");
    if (reinterpret_cast<uintptr_t>(out_rgbt) % 16) return fail(NSL_ERR_INVALID_ARG, "out_rgbt must be 16-B aligned");
    return NSL_OK;
}

static nsl_status batch_impl(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                             const nsl_camera* cams, const nsl_light* lights, int32_t n_lights, int32_t light_mode,
                             const nsl_medium* med, const nsl_march* m, const uint32_t* frame_ids, int32_t F,
                             float* out_rgbt, float* out_depth, uint32_t* out_debug, unsigned long long* counters,
                             nsl_stream stream) {
    g_err.clear();
    if (nsl_status st = check_outputs(out_rgbt, out_depth)) return st;
    Prepared P;
    if (nsl_status st = prepare(vols, n_vols, frame_vol, cams, lights, n_lights, light_mode, med, m, frame_ids, F, P))
        return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Workspace ws;
    if (nsl_status st = build_frames(P.frames, lights, n_lights, P.mc, true, s, ws)) return st;
    void* tvws = nullptr;
    cudaError_t e = cudaSuccess;
    if (P.tv_slots) e = pool_malloc(&tvws, align_up(P.tv_params_bytes(), 256) + P.tv_buf_bytes(), s);
    if (e == cudaSuccess)
        e = run_march(P, ws.params, ws.cull, static_cast<TvParams*>(tvws),
                      reinterpret_cast<float2*>(static_cast<char*>(tvws) + align_up(P.tv_params_bytes(), 256)),
                      out_rgbt, out_depth, out_debug, counters, s);
    if (tvws) cudaFreeAsync(tvws, s);
    cudaError_t e2 = cudaFreeAsync(ws.base, s);
    if (e != cudaSuccess) return cuda_fail(e, "march_kernel launch");
    if (e2 != cudaSuccess) return cuda_fail(e2, "cudaFreeAsync(frame tables)");
    return NSL_OK;
}

nsl_status nsl_guiding_map_batch(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                                 const nsl_camera* cams, const nsl_light* lights, int32_t n_lights, int32_t light_mode,
                                 const nsl_medium* med, const nsl_march* m, const uint32_t* frame_ids, int32_t F,
                                 float* out_rgbt, float* out_depth, uint32_t* out_debug, nsl_stream stream) {
    return batch_impl(vols, n_vols, frame_vol, cams, lights, n_lights, light_mode, med, m, frame_ids, F, out_rgbt,
                      out_depth, out_debug, nullptr, stream);
}

nsl_status nsl_guiding_map_batch_counted(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                                         const nsl_camera* cams, const nsl_light* lights, int32_t n_lights,
                                         int32_t light_mode, const nsl_medium* med, const nsl_march* m,
                                         const uint32_t* frame_ids, int32_t F, float* out_rgbt, float* out_depth,
                                         uint64_t* counters, nsl_stream stream) {
    if (!counters) {
        g_err = "counters is NULL";
        return NSL_ERR_INVALID_ARG;
    }
    NSL_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(uint64_t), reinterpret_cast<cudaStream_t>(stream)),
             "cudaMemsetAsync(counters)");
    return batch_impl(vols, n_vols, frame_vol, cams, lights, n_lights, light_mode, med, m, frame_ids, F, out_rgbt,
                      out_depth, nullptr, reinterpret_cast<unsigned long long*>(counters), stream);
}

nsl_status nsl_guiding_map(const nsl_volume* vol, const nsl_camera* cam, const nsl_light* lights, int32_t n_lights,
                           int32_t light_mode, const nsl_medium* med, const nsl_march* m, uint32_t frame_id,
                           float* out_rgbt, float* out_depth, uint32_t* out_debug, nsl_stream stream) {
    if (!vol || !cam) {
        g_err = "NULL volume/camera";
        return NSL_ERR_INVALID_ARG;
    }
    const int32_t zero = 0;
    return nsl_guiding_map_batch(&vol, 1, &zero, cam, lights, n_lights, light_mode, med, m, &frame_id, 1, out_rgbt,
                                 out_depth, out_debug, stream);
}

// host_half: outputs are packed to fp16 on the device (pack_half_kernel) before the download
static nsl_status host_impl(const nsl_grid_desc* g, const float* host_density, int32_t layout, const nsl_camera* cams,
                            const nsl_light* lights, int32_t n_lights, int32_t light_mode, const nsl_medium* med,
                            const nsl_march* m, const uint32_t* frame_ids, int32_t F, void* host_rgbt, void* host_depth,
                            bool host_half, nsl_stream stream) {
    g_err.clear();
    if (nsl_status st = check_grid(g)) return st;
    layout = resolve_layout(g, layout);
    if (nsl_status st = check_layout(layout)) return st;
    if (!host_density || !cams || !host_rgbt || !host_depth) return fail(NSL_ERR_INVALID_ARG, "NULL host buffer");
    if (F < 1) return fail(NSL_ERR_INVALID_ARG, "F must be >= 1");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t vb = nsl_volume_bytes(g, layout);
    const size_t npix = (size_t)F * cams[0].width * cams[0].height;
    void *vstore = nullptr, *dout = nullptr;
    NSL_CUDA(pool_malloc(&vstore, vb, s), "cudaMallocAsync(volume)");
    cudaError_t e = pool_malloc(&dout, npix * (host_half ? 30 : 20), s);
    if (e != cudaSuccess) {
        cudaFreeAsync(vstore, s);
        return cuda_fail(e, "cudaMallocAsync(outputs)");
    }
    float* d_rgbt = static_cast<float*>(dout);
    float* d_depth = d_rgbt + npix * 4;
    uint16_t* h_rgbt = reinterpret_cast<uint16_t*>(d_depth + npix);      // fp16 staging (host_half)
    uint16_t* h_depth = h_rgbt + npix * 4;
    nsl_volume* vol = nullptr;
    std::vector<int32_t> fv((size_t)F, 0);
    nsl_status st = volume_upload_impl(g, host_density, 0, layout, vstore, vb, stream, &vol, false);
    // Frame chunks: chunk c marches on `stream` while chunk c-1's results stream back to the
    // host on a side stream (PCIe D2H overlaps the march; the copies dominate for fp32 maps).
    cudaStream_t side = nullptr;
    std::vector<cudaEvent_t> evs;
    const size_t npf = (size_t)cams[0].width * cams[0].height;
    int want = 8;                                 // chunks (NSL_HOST_CHUNKS overrides)
    if (const char* ev = getenv("NSL_HOST_CHUNKS")) want = atoi(ev) > 0 ? atoi(ev) : 8;
    const int nchunks = F < want ? F : want, per = (F + nchunks - 1) / nchunks;
    if (st == NSL_OK) {
        e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
        if (e != cudaSuccess) st = cuda_fail(e, "cudaStreamCreate(side)");
    }
    const nsl_volume* vp = vol;
    for (int f0 = 0; st == NSL_OK && f0 < F; f0 += per) {
        const int n = F - f0 < per ? F - f0 : per;
        st = batch_impl(&vp, 1, fv.data(), cams + f0, lights ? lights + (size_t)f0 * n_lights : nullptr, n_lights,
                        light_mode, med, m, frame_ids ? frame_ids + f0 : nullptr, n, d_rgbt + (size_t)f0 * npf * 4,
                        d_depth + (size_t)f0 * npf, nullptr, nullptr, stream);
        if (st != NSL_OK) break;
        cudaEvent_t ev = nullptr;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) {
            evs.push_back(ev);
            e = cudaEventRecord(ev, s);
        }
        if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev, 0);
        const size_t p0 = (size_t)f0 * npf, pn = (size_t)n * npf;
        if (host_half) {                          // pack on the side stream, then download 10 B/pixel
            if (e == cudaSuccess) e = launch_pack_half(d_rgbt + p0 * 4, d_depth + p0, h_rgbt + p0 * 4, h_depth + p0, pn, side);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(static_cast<uint16_t*>(host_rgbt) + p0 * 4, h_rgbt + p0 * 4, pn * 8,
                                    cudaMemcpyDeviceToHost, side);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(static_cast<uint16_t*>(host_depth) + p0, h_depth + p0, pn * 2,
                                    cudaMemcpyDeviceToHost, side);
        } else {
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(static_cast<float*>(host_rgbt) + p0 * 4, d_rgbt + p0 * 4, pn * 16,
                                    cudaMemcpyDeviceToHost, side);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(static_cast<float*>(host_depth) + p0, d_depth + p0, pn * 4,
                                    cudaMemcpyDeviceToHost, side);
        }
        if (e != cudaSuccess) st = cuda_fail(e, "result download");
    }
    if (side) {                                   // `stream` resumes after the last copy
        cudaEvent_t done = nullptr;
        if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) == cudaSuccess) {
            evs.push_back(done);
            cudaEventRecord(done, side);
            cudaStreamWaitEvent(s, done, 0);
        } else {
            cudaStreamSynchronize(side);
        }
    }
    unsigned long long n_invalid = 0;
    if (vol) cudaMemcpyAsync(&n_invalid, vol->invalid, sizeof n_invalid, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(dout, s);
    cudaFreeAsync(vstore, s);
    nsl_volume_release(vol);
    cudaError_t es = cudaStreamSynchronize(s);
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
    if (side) cudaStreamDestroy(side);
    if (st != NSL_OK) return st;
    if (es != cudaSuccess) return cuda_fail(es, "cudaStreamSynchronize");
    if (n_invalid) return fail(NSL_ERR_INVALID_ARG, "density has %llu non-finite or negative values", n_invalid);
    return NSL_OK;
}

nsl_status nsl_guiding_map_host(const nsl_grid_desc* g, const float* host_density, int32_t layout,
                                const nsl_camera* cams, const nsl_light* lights, int32_t n_lights, int32_t light_mode,
                                const nsl_medium* med, const nsl_march* m, const uint32_t* frame_ids, int32_t F,
                                float* host_rgbt, float* host_depth, nsl_stream stream) {
    return host_impl(g, host_density, layout, cams, lights, n_lights, light_mode, med, m, frame_ids, F, host_rgbt,
                     host_depth, false, stream);
}

nsl_status nsl_guiding_map_host_f16(const nsl_grid_desc* g, const float* host_density, int32_t layout,
                                    const nsl_camera* cams, const nsl_light* lights, int32_t n_lights,
                                    int32_t light_mode, const nsl_medium* med, const nsl_march* m,
                                    const uint32_t* frame_ids, int32_t F, uint16_t* host_rgbt_h,
                                    uint16_t* host_depth_h, nsl_stream stream) {
    return host_impl(g, host_density, layout, cams, lights, n_lights, light_mode, med, m, frame_ids, F, host_rgbt_h,
                     host_depth_h, true, stream);
}

// Animated volumes: frame f's density is laid out into its own storage and marched with its
// own camera.  Chunks of frames: the layouts of chunk c+1 build on a side stream while chunk c
// marches on `stream`; an event per chunk orders its march after its builds, and `stream`
// waits for the side stream at the end, so everything is ordered on `stream` on return.
nsl_status nsl_guiding_map_animated(const nsl_grid_desc* g, const float* const* densities, int32_t layout,
                                    void* const* storage, size_t storage_bytes, const nsl_camera* cams,
                                    const nsl_light* lights, int32_t n_lights, int32_t light_mode,
                                    const nsl_medium* med, const nsl_march* m, const uint32_t* frame_ids, int32_t F,
                                    int32_t chunk, float* out_rgbt, float* out_depth, uint64_t* n_invalid,
                                    nsl_stream stream) {
    g_err.clear();
    if (nsl_status st = check_grid(g)) return st;
    layout = resolve_layout(g, layout, true);
    if (nsl_status st = check_layout(layout)) return st;
    if (!densities || !storage || !cams) return fail(NSL_ERR_INVALID_ARG, "NULL densities/storage/cameras");
    if (F < 1) return fail(NSL_ERR_INVALID_ARG, "F must be >= 1");
    if (chunk < 0) return fail(NSL_ERR_INVALID_ARG, "chunk must be >= 0");
    if (nsl_status st = check_outputs(out_rgbt, out_depth)) return st;
    // every argument is checked (host only) before anything is enqueued
    std::vector<nsl_volume*> vols((size_t)F, nullptr);
    auto release_all = [&]() {
        for (nsl_volume* v : vols) nsl_volume_release(v);
    };
    for (int f = 0; f < F; ++f) {
        nsl_status st = densities[f] ? volume_handle(g, layout, storage[f], storage_bytes, &vols[f])
                                     : fail(NSL_ERR_INVALID_ARG, "NULL density of frame %d", f);
        if (st != NSL_OK) {
            release_all();
            return st;
        }
    }
    std::vector<int32_t> fv((size_t)F);
    for (int f = 0; f < F; ++f) fv[f] = f;
    Prepared P;
    const nsl_volume* const* vp = const_cast<const nsl_volume* const*>(vols.data());
    if (nsl_status st = prepare(vp, F, fv.data(), cams, lights, n_lights, light_mode, med, m, frame_ids, F, P)) {
        release_all();
        return st;
    }
    const int per = chunk > 0 ? chunk : 6;       // C4 is insensitive to it (3..60)
    const size_t npf = (size_t)cams[0].width * cams[0].height;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream), side = nullptr;
    std::vector<cudaEvent_t> evs;
    auto event_on = [&](cudaStream_t from, cudaStream_t to) -> cudaError_t {
        cudaEvent_t ev = nullptr;
        cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
        evs.push_back(ev);
        e = cudaEventRecord(ev, from);
        return e == cudaSuccess ? cudaStreamWaitEvent(to, ev, 0) : e;
    };
    nsl_status st = NSL_OK;
    cudaError_t e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    if (e != cudaSuccess) st = cuda_fail(e, "cudaStreamCreate(side)");
    if (st == NSL_OK && (e = event_on(s, side)) != cudaSuccess)   // builds follow earlier work on `stream`
        st = cuda_fail(e, "stream ordering");
    // frame tables of all F frames in one upload; per chunk only frame setup + march
    Workspace ws;
    void* tvws = nullptr;
    const size_t tiles = march_cull_bytes(1, P.W, P.H) / sizeof(TileCull);
    Prepared Pc = P;                             // a chunk's view of P (F = frames of the chunk)
    Pc.tv_group = P.tv_group < per ? P.tv_group : per;
    if (st == NSL_OK) st = upload_frames(P.frames, lights, n_lights, true, s, ws);
    if (st == NSL_OK && P.tv_slots) {
        Pc.F = per;
        e = pool_malloc(&tvws, align_up(Pc.tv_params_bytes(), 256) + Pc.tv_buf_bytes(), s);
        if (e != cudaSuccess) st = cuda_fail(e, "cudaMallocAsync(TV workspace)");
    }
    for (int f0 = 0; st == NSL_OK && f0 < F; f0 += per) {
        const int n = F - f0 < per ? F - f0 : per;
        for (int f = f0; e == cudaSuccess && f < f0 + n; ++f) e = enqueue_build(vols[f], densities[f], side);
        if (e != cudaSuccess) {
            st = cuda_fail(e, "volume build launch");
            break;
        }
        if ((e = event_on(side, s)) != cudaSuccess) {
            st = cuda_fail(e, "chunk ordering");
            break;
        }
        Pc.F = n;
        e = launch_frame_setup(ws.in + f0, ws.lights + (size_t)f0 * n_lights, n, P.mc, ws.params + f0, s);
        if (e == cudaSuccess)
            e = run_march(Pc, ws.params + f0, ws.cull + (size_t)f0 * tiles, static_cast<TvParams*>(tvws),
                          reinterpret_cast<float2*>(static_cast<char*>(tvws) + align_up(Pc.tv_params_bytes(), 256)),
                          out_rgbt + (size_t)f0 * npf * 4, out_depth + (size_t)f0 * npf, nullptr, nullptr, s);
        if (e != cudaSuccess) st = cuda_fail(e, "march launch");
    }
    if (tvws) cudaFreeAsync(tvws, s);
    if (ws.base) cudaFreeAsync(ws.base, s);
    if (side) {
        e = event_on(side, s);                   // `stream` resumes after every build
        if (e != cudaSuccess) cudaStreamSynchronize(side);
    }
    unsigned long long* counts = nullptr;
    if (st == NSL_OK && n_invalid) {             // the build kernels' invalid-voxel counters
        e = cudaMallocHost(&counts, sizeof(unsigned long long) * F);
        for (int f = 0; e == cudaSuccess && f < F; ++f)
            e = cudaMemcpyAsync(counts + f, vols[f]->invalid, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = cuda_fail(e, "invalid-voxel counters");
        uint64_t tot = 0;
        for (int f = 0; st == NSL_OK && f < F; ++f) tot += counts[f];
        *n_invalid = tot;
    }
    if (counts) cudaFreeHost(counts);
    release_all();
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);   // released once they complete
    if (side) cudaStreamDestroy(side);
    return st;
}

struct nsl_plan {
    Prepared P;                 // frames vector cleared after upload
    void* dev = nullptr;        // FrameIn[F] | lights[F*nl] | FrameParams[F]
    FrameIn* in = nullptr;
    nsl_light* lights = nullptr;
    FrameParams* params = nullptr;
    TileCull* cull = nullptr;
    TvParams* tvp = nullptr;     // NEXT-4 workspace (light_model TV)
    float2* tvbuf = nullptr;
};

nsl_status nsl_plan_create(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                           const nsl_camera* cams, const nsl_light* lights, int32_t n_lights, int32_t light_mode,
                           const nsl_medium* med, const nsl_march* m, const uint32_t* frame_ids, int32_t F,
                           nsl_stream stream, nsl_plan** out) {
    g_err.clear();
    if (!out) return fail(NSL_ERR_INVALID_ARG, "NULL out");
    nsl_plan* p = new nsl_plan;
    if (nsl_status st = prepare(vols, n_vols, frame_vol, cams, lights, n_lights, light_mode, med, m, frame_ids, F, p->P)) {
        delete p;
        return st;
    }
    const size_t b_in = align_up(sizeof(FrameIn) * F, 256);
    const size_t b_l = align_up(sizeof(nsl_light) * (size_t)F * n_lights, 256);
    const size_t b_p = align_up(sizeof(FrameParams) * F, 256);
    const size_t b_c = align_up(march_cull_bytes(F, p->P.W, p->P.H), 256);
    const size_t b_tp = align_up(p->P.tv_params_bytes(), 256);
    cudaError_t e = cudaMalloc(&p->dev, b_in + b_l + b_p + b_c + b_tp + p->P.tv_buf_bytes());
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "cudaMalloc(plan)");
    }
    p->in = reinterpret_cast<FrameIn*>(p->dev);
    p->lights = reinterpret_cast<nsl_light*>(static_cast<char*>(p->dev) + b_in);
    p->params = reinterpret_cast<FrameParams*>(static_cast<char*>(p->dev) + b_in + b_l);
    p->cull = reinterpret_cast<TileCull*>(static_cast<char*>(p->dev) + b_in + b_l + b_p);
    p->tvp = reinterpret_cast<TvParams*>(static_cast<char*>(p->dev) + b_in + b_l + b_p + b_c);
    p->tvbuf = reinterpret_cast<float2*>(static_cast<char*>(p->dev) + b_in + b_l + b_p + b_c + b_tp);
    std::vector<char> host(b_in + b_l);
    memcpy(host.data(), p->P.frames.data(), sizeof(FrameIn) * F);
    memcpy(host.data() + b_in, lights, sizeof(nsl_light) * (size_t)F * n_lights);
    e = cudaMemcpyAsync(p->dev, host.data(), host.size(), cudaMemcpyHostToDevice, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) {
        cudaFree(p->dev);
        delete p;
        return cuda_fail(e, "plan upload");
    }
    p->P.frames.clear();
    p->P.frames.shrink_to_fit();
    *out = p;
    return NSL_OK;
}

nsl_status nsl_plan_execute(const nsl_plan* p, float* out_rgbt, float* out_depth, uint32_t* out_debug,
                            uint64_t* counters, nsl_stream stream) {
    g_err.clear();
    if (!p) return fail(NSL_ERR_INVALID_ARG, "NULL plan");
    if (nsl_status st = check_outputs(out_rgbt, out_depth)) return st;
    if (out_debug && counters) return fail(NSL_ERR_INVALID_ARG, "debug and counters are exclusive");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (counters) NSL_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(uint64_t), s), "cudaMemsetAsync(counters)");
    NSL_CUDA(launch_frame_setup(p->in, p->lights, p->P.F, p->P.mc, p->params, s), "frame_setup_kernel launch");
    NSL_CUDA(run_march(p->P, p->params, p->cull, p->tvp, p->tvbuf, out_rgbt, out_depth, out_debug,
                       reinterpret_cast<unsigned long long*>(counters), s),
             "march_kernel launch");
    return NSL_OK;
}

nsl_status nsl_plan_destroy(nsl_plan* p) {
    if (!p) return NSL_OK;
    cudaError_t e = cudaFree(p->dev);
    delete p;
    return e == cudaSuccess ? NSL_OK : cuda_fail(e, "cudaFree(plan)");
}

// ------------------------------------------------------------------ NEXT-1 six-way bake
static nsl_status check_bake(const nsl_bake* b) {
    if (!b) return fail(NSL_ERR_INVALID_ARG, "bake params are NULL");
    if (b->spp < 1 || b->spp > (1 << 20)) return fail(NSL_ERR_INVALID_ARG, "spp must be in [1, 2^20]");
    if (!(b->step > 0.0f) || !std::isfinite(b->step)) return fail(NSL_ERR_INVALID_ARG, "bake step must be > 0");
    if (!(b->light_step > 0.0f) || !std::isfinite(b->light_step))
        return fail(NSL_ERR_INVALID_ARG, "bake light_step must be > 0");
    if (b->max_steps < 0 || b->max_steps > (1 << 24)) return fail(NSL_ERR_INVALID_ARG, "max_steps out of range");
    if (!(b->t_min >= 0.0f && b->t_min < 1.0f)) return fail(NSL_ERR_INVALID_ARG, "t_min must be in [0,1)");
    return NSL_OK;
}

nsl_status nsl_sixway_bake(const nsl_volume* const* vols, int32_t n_vols, const int32_t* frame_vol,
                           const nsl_camera* cams, const nsl_medium* med, const nsl_bake* b,
                           const uint32_t* frame_ids, int32_t F, float* out, uint64_t* counters,
                           nsl_stream stream) {
    g_err.clear();
    if (nsl_status st = check_bake(b)) return st;
    if (!out) return fail(NSL_ERR_INVALID_ARG, "NULL output");
    if (reinterpret_cast<uintptr_t>(out) % 16) return fail(NSL_ERR_INVALID_ARG, "out must be 16-B aligned");
    if (F < 1 || F > 65535) return fail(NSL_ERR_INVALID_ARG, "F must be in [1, 65535]");
    // the six axis lights are fixed; the march constants carry only the camera/volume part
    std::vector<nsl_light> dummy((size_t)F, nsl_light{{1.0f, 0.0f, 0.0f}, {1.0f, 1.0f, 1.0f}});
    nsl_march m{};
    m.step = b->step;
    m.light_step = b->light_step;
    m.max_steps = b->max_steps;
    m.t_min = b->t_min;
    m.seed = b->seed;
    Prepared P;
    if (nsl_status st = prepare(vols, n_vols, frame_vol, cams, dummy.data(), 1, NSL_LIGHTS_EXPLICIT, med, &m,
                                frame_ids, F, P))
        return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Workspace ws;
    if (nsl_status st = build_frames(P.frames, dummy.data(), 1, P.mc, false, s, ws)) return st;
    BakeFrame* bf = nullptr;
    cudaError_t e = pool_malloc(&bf, sizeof(BakeFrame) * F, s);
    if (e == cudaSuccess) e = launch_bake_setup(ws.in, ws.params, F, b->light_step, med->hg_g, bf, s);
    if (e == cudaSuccess && counters) e = cudaMemsetAsync(counters, 0, sizeof(uint64_t), s);
    if (e == cudaSuccess) {
        BakeConst bc;
        bc.hb = b->step;
        bc.hbl = b->light_step;
        bc.kappa = med->extinction;
        bc.alpha = med->albedo;
        bc.g = med->hg_g;
        bc.t_min = b->t_min;
        bc.spp = b->spp;
        bc.Ncap = b->max_steps > 0 ? b->max_steps : (1 << 24);
        bc.seed_lo = (uint32_t)(b->seed & 0xffffffffu);
        bc.seed_hi = (uint32_t)(b->seed >> 32);
        bc.counters = reinterpret_cast<unsigned long long*>(counters);
        e = launch_bake(ws.params, bf, bc, F, P.W, P.H, P.proj, P.layout, reinterpret_cast<float4*>(out), s);
    }
    if (bf) cudaFreeAsync(bf, s);
    cudaFreeAsync(ws.base, s);
    if (e != cudaSuccess) return cuda_fail(e, "six-way bake launch");
    return NSL_OK;
}

nsl_status nsl_relight(const nsl_camera* cams, int32_t F, const float* maps, const float* depth,
                       const nsl_light* lights, int32_t n_lights, const float bg[3], const float emis[3],
                       const nsl_camera* shadow_cams, const float* const* shadow_maps, float bias,
                       float* out, nsl_stream stream) {
    g_err.clear();
    if (F < 1 || F > (1 << 20)) return fail(NSL_ERR_INVALID_ARG, "F out of range");
    if (!cams || !maps || !lights || !bg || !emis || !out) return fail(NSL_ERR_INVALID_ARG, "NULL argument");
    if (n_lights < 1 || n_lights > 4) return fail(NSL_ERR_INVALID_ARG, "n_lights must be in [1,4]");
    if (reinterpret_cast<uintptr_t>(maps) % 16 || reinterpret_cast<uintptr_t>(out) % 16)
        return fail(NSL_ERR_INVALID_ARG, "maps/out must be 16-B aligned");
    if (!(bias >= 0.0f) || !std::isfinite(bias)) return fail(NSL_ERR_INVALID_ARG, "bias must be finite and >= 0");
    if (!finite3(bg) || !finite3(emis)) return fail(NSL_ERR_INVALID_ARG, "bg/emis must be finite");
    const int W = cams[0].width, H = cams[0].height;
    std::vector<RelightIn> in((size_t)F);
    bool any_shadow = false;
    for (int f = 0; f < F; ++f) {
        if (nsl_status st = check_camera(&cams[f], f)) return st;
        if (cams[f].width != W || cams[f].height != H) return fail(NSL_ERR_INVALID_ARG, "camera[%d]: size differs", f);
        if (nsl_status st = check_lights(lights + (size_t)f * n_lights, n_lights, NSL_LIGHTS_EXPLICIT, f)) return st;
        RelightIn& ri = in[f];
        memset(&ri, 0, sizeof ri);
        ri.cam = cams[f];
        for (int l = 0; l < n_lights; ++l) {
            ri.lights[l] = lights[(size_t)f * n_lights + l];
            const float* sm = shadow_maps ? shadow_maps[(size_t)f * n_lights + l] : nullptr;
            if (sm) {
                if (!depth) return fail(NSL_ERR_INVALID_ARG, "shadow maps need the depth map");
                if (!shadow_cams) return fail(NSL_ERR_INVALID_ARG, "shadow maps need shadow cameras");
                const nsl_camera& sc = shadow_cams[(size_t)f * n_lights + l];
                if (nsl_status st = check_camera(&sc, f)) return st;
                if (sc.projection != 0) return fail(NSL_ERR_UNSUPPORTED, "shadow cameras must be orthographic");
                ri.shadow_cam[l] = sc;
                ri.shadow_map[l] = sm;
                any_shadow = true;
            }
        }
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    void* ws = nullptr;
    const size_t b_in = align_up(sizeof(RelightIn) * F, 256);
    NSL_CUDA(pool_malloc(&ws, b_in + sizeof(RelightFrame) * F, s), "cudaMallocAsync(relight tables)");
    cudaError_t e = cudaMemcpyAsync(ws, in.data(), sizeof(RelightIn) * F, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        RelightConst rc;
        rc.F = F;
        rc.W = W;
        rc.H = H;
        rc.n_lights = n_lights;
        rc.any_shadow = any_shadow ? 1 : 0;
        rc.bias = bias;
        for (int a = 0; a < 3; ++a) {
            rc.bg[a] = bg[a];
            rc.emis[a] = emis[a];
        }
        e = launch_relight(static_cast<const RelightIn*>(ws), F, n_lights,
                           reinterpret_cast<RelightFrame*>(static_cast<char*>(ws) + b_in), rc,
                           reinterpret_cast<const float4*>(maps), depth, reinterpret_cast<float4*>(out), s);
    }
    cudaFreeAsync(ws, s);
    if (e != cudaSuccess) return cuda_fail(e, "relight launch");
    return NSL_OK;
}

nsl_status nsl_debug_bake_lights(const nsl_grid_desc* g, const nsl_camera* cam, float Lg[6][3], float Ln[6][3],
                                 nsl_stream stream) {
    g_err.clear();
    if (nsl_status st = check_grid(g)) return st;
    if (!cam || !Lg || !Ln) return fail(NSL_ERR_INVALID_ARG, "NULL camera/output");
    if (nsl_status st = check_camera(cam, 0)) return st;
    std::vector<FrameIn> frames(1);
    memset(frames.data(), 0, sizeof(FrameIn));
    frames[0].cam = *cam;
    frames[0].vol.nx = g->nx;
    frames[0].vol.ny = g->ny;
    frames[0].vol.nz = g->nz;
    frames[0].vol.layout = kQuadF32;
    for (int a = 0; a < 3; ++a) frames[0].vol.origin[a] = g->origin[a];
    frames[0].vol.dx = g->voxel_width;
    nsl_light dummy{{1.0f, 0.0f, 0.0f}, {1.0f, 1.0f, 1.0f}};
    nsl_medium med{0.0f, 1.0f, 0.0f};
    nsl_march m{};
    m.step = g->voxel_width;
    const MarchConst mc = make_const(1, NSL_LIGHTS_EXPLICIT, &med, &m);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Workspace ws;
    if (nsl_status st = build_frames(frames, &dummy, 1, mc, false, s, ws)) return st;
    BakeFrame* bf = nullptr;
    BakeFrame h;
    cudaError_t e = pool_malloc(&bf, sizeof(BakeFrame), s);
    if (e == cudaSuccess) e = launch_bake_setup(ws.in, ws.params, 1, m.step, 0.0f, bf, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, bf, sizeof h, cudaMemcpyDeviceToHost, s);
    if (bf) cudaFreeAsync(bf, s);
    cudaFreeAsync(ws.base, s);
    if (e != cudaSuccess) return cuda_fail(e, "bake light setup");
    NSL_CUDA(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    memcpy(Lg, h.Lg, sizeof h.Lg);
    memcpy(Ln, h.Ln, sizeof h.Ln);
    return NSL_OK;
}

nsl_status nsl_debug_frame_constants(const nsl_grid_desc* g, const nsl_camera* cam, const nsl_light* lights,
                                     int32_t n_lights, int32_t light_mode, const nsl_medium* med, const nsl_march* m,
                                     nsl_frame_constants* out, nsl_stream stream) {
    g_err.clear();
    if (nsl_status st = check_grid(g)) return st;
    if (!cam || !out) return fail(NSL_ERR_INVALID_ARG, "NULL camera/out");
    if (nsl_status st = check_camera(cam, 0)) return st;
    if (nsl_status st = check_common(lights, n_lights, light_mode, med, m)) return st;
    if (nsl_status st = check_lights(lights, n_lights, light_mode, 0)) return st;
    std::vector<FrameIn> frames(1);
    memset(frames.data(), 0, sizeof(FrameIn));
    frames[0].cam = *cam;
    frames[0].vol.nx = g->nx;
    frames[0].vol.ny = g->ny;
    frames[0].vol.nz = g->nz;
    frames[0].vol.layout = kQuadF32;
    for (int a = 0; a < 3; ++a) frames[0].vol.origin[a] = g->origin[a];
    frames[0].vol.dx = g->voxel_width;
    const MarchConst mc = make_const(n_lights, light_mode, med, m);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Workspace ws;
    if (nsl_status st = build_frames(frames, lights, n_lights, mc, false, s, ws)) return st;
    FrameParams p;
    cudaError_t e = cudaMemcpyAsync(&p, ws.params, sizeof p, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(ws.base, s);
    if (e != cudaSuccess) return cuda_fail(e, "frame constants download");
    NSL_CUDA(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    out->inv_dx = p.inv_dx;
    memcpy(out->B, p.B, sizeof p.B);
    memcpy(out->Ex, p.Ex, sizeof p.Ex);
    memcpy(out->Ey, p.Ey, sizeof p.Ey);
    memcpy(out->Dg, p.Dg, sizeof p.Dg);
    memcpy(out->Oe, p.Oe, sizeof p.Oe);
    memcpy(out->F0, p.F0, sizeof p.F0);
    memcpy(out->fwd, p.fwd, sizeof p.fwd);
    memcpy(out->Ln, p.Ln, sizeof p.Ln);
    memcpy(out->Lg, p.Lg, sizeof p.Lg);
    memcpy(out->P, p.P, sizeof p.P);
    out->front_identity_ok = p.front_ok;
    return NSL_OK;
}

nsl_status nsl_guide_lights(const nsl_camera* cam, const float axis[3], const float rgb[3], nsl_light out[3],
                            nsl_stream stream) {
    g_err.clear();
    if (!cam || !out) return fail(NSL_ERR_INVALID_ARG, "NULL camera/out");
    if (axis && !finite3(axis)) return fail(NSL_ERR_INVALID_ARG, "axis must be finite");
    if (rgb && (!finite3(rgb) || rgb[0] < 0.0f || rgb[1] < 0.0f || rgb[2] < 0.0f))
        return fail(NSL_ERR_INVALID_ARG, "rgb must be finite and >= 0");
    const nsl_grid_desc g = {1, 1, 1, {0.0f, 0.0f, 0.0f}, 1.0f};
    const nsl_medium med = {1.0f, 1.0f, 0.0f};
    nsl_march m;
    memset(&m, 0, sizeof m);
    m.step = 1.0f;
    m.t_min = 1e-4f;
    m.guide_axis[0] = axis ? axis[0] : 0.0f;
    m.guide_axis[1] = axis ? axis[1] : 0.0f;
    m.guide_axis[2] = axis ? axis[2] : 1.0f;
    nsl_light in[3];
    for (int l = 0; l < 3; ++l)
        for (int a = 0; a < 3; ++a) {
            in[l].to_light[a] = a == 0 ? 1.0f : 0.0f;      // ignored in guide mode
            in[l].rgb[a] = rgb ? rgb[a] : 1.0f;
        }
    nsl_frame_constants fc;
    if (nsl_status st = nsl_debug_frame_constants(&g, cam, in, 3, NSL_LIGHTS_GUIDE, &med, &m, &fc, stream)) return st;
    for (int l = 0; l < 3; ++l) {
        memcpy(out[l].to_light, fc.Ln[l], sizeof out[l].to_light);
        memcpy(out[l].rgb, in[l].rgb, sizeof out[l].rgb);
    }
    return NSL_OK;
}

nsl_status nsl_bench_l1_gather(const nsl_volume* vol, int32_t waves, int32_t reps, float* sink, size_t sink_floats,
                               uint64_t* samples, nsl_stream stream) {
    g_err.clear();
    if (!vol || !sink || !samples) return fail(NSL_ERR_INVALID_ARG, "NULL volume/sink/samples");
    if (waves < 1 || reps < 1) return fail(NSL_ERR_INVALID_ARG, "waves and reps must be >= 1");
    const nsl_grid_desc& g = vol->g;
    if (g.nx < 16 || g.ny < 16 || g.nz < 16) return fail(NSL_ERR_INVALID_ARG, "the volume must be at least 16^3");
    int dev = 0, sms = 0;
    NSL_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    NSL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    const int per_sm = l1_gather_max_blocks_per_sm(vol->layout);
    const size_t blocks = (size_t)sms * (per_sm > 0 ? per_sm : 1) * waves;
    const size_t threads = blocks * l1_gather_threads();
    if (sink_floats < threads) return fail(NSL_ERR_INVALID_ARG, "sink needs %zu floats", threads);
    FrameParams p;
    memset(&p, 0, sizeof p);
    p.data = vol->data;
    p.layout = vol->layout;
    layout_strides(vol->layout, g.nx, g.ny, p.sy, p.sz);
    p.supp[0] = (float)(g.nx + 1);
    p.supp[1] = (float)(g.ny + 1);
    p.supp[2] = (float)(g.nz + 1);
    p.occ = vol->occ;
    p.occ_shift = vol->og.shift;
    p.occ_nbx = vol->og.nbx;
    p.occ_nby = vol->og.nby;
    p.slab_off = vol->og.words;
    NSL_CUDA(launch_l1_gather(p, (int)blocks, reps, sink, reinterpret_cast<cudaStream_t>(stream)),
             "l1_gather_kernel launch");
    *samples = (uint64_t)threads * reps * l1_gather_line();
    return NSL_OK;
}

nsl_status nsl_bench_l1_peak(const float* buf, size_t buf_floats, const int32_t* lane_off, int32_t max_off,
                             int64_t stride_elems, int64_t span_elems, int32_t waves, int32_t reps, float* sink,
                             size_t sink_floats, uint64_t* bytes, nsl_stream stream) {
    g_err.clear();
    if (!buf || !lane_off || !sink || !bytes) return fail(NSL_ERR_INVALID_ARG, "NULL buf/lane_off/sink/bytes");
    if (waves < 1 || reps < 1 || max_off < 0 || stride_elems < 0 || span_elems < 1)
        return fail(NSL_ERR_INVALID_ARG, "bad waves/reps/max_off/stride/span");
    if (reinterpret_cast<uintptr_t>(buf) % 32) return fail(NSL_ERR_INVALID_ARG, "buf must be 32-B aligned");
    // every load stays inside buf: (span - 1 + max_off + 1) elements of 8 floats
    if ((uint64_t)(span_elems + max_off) * 8 > buf_floats)
        return fail(NSL_ERR_INVALID_ARG, "buf needs %lld floats", (long long)(span_elems + max_off) * 8);
    int dev = 0, sms = 0;
    NSL_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    NSL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    const int per_sm = l1_peak_max_blocks_per_sm();
    const size_t blocks = (size_t)sms * (per_sm > 0 ? per_sm : 1) * waves;
    const size_t threads = blocks * l1_peak_threads();
    if (sink_floats < threads) return fail(NSL_ERR_INVALID_ARG, "sink needs %zu floats", threads);
    NSL_CUDA(launch_l1_peak(buf, lane_off, (long long)(stride_elems % span_elems), (long long)span_elems,
                            (int)blocks, reps, sink, reinterpret_cast<cudaStream_t>(stream)),
             "l1_peak_kernel launch");
    *bytes = (uint64_t)threads * reps * l1_peak_patterns() * 32;
    return NSL_OK;
}

nsl_status nsl_debug_tex_filter(const nsl_grid_desc* g, const float* density, const float* positions, int32_t n,
                                float* out, nsl_stream stream) {
    g_err.clear();
    if (nsl_status st = check_grid(g)) return st;
    if (!density || !positions || !out || n < 0) return fail(NSL_ERR_INVALID_ARG, "bad arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int px = g->nx + 2, py = g->ny + 2, pz = g->nz + 2;
    // the padded grid (zero apron, C1) on the host, then a float cudaArray with linear filtering
    std::vector<float> pad((size_t)px * py * pz, 0.0f);
    std::vector<float> raw((size_t)g->nx * g->ny * g->nz);
    NSL_CUDA(cudaMemcpyAsync(raw.data(), density, raw.size() * sizeof(float), cudaMemcpyDeviceToHost, s), "density read");
    NSL_CUDA(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    for (int k = 0; k < g->nz; ++k)
        for (int j = 0; j < g->ny; ++j)
            for (int i = 0; i < g->nx; ++i)
                pad[((size_t)(k + 1) * py + (j + 1)) * px + (i + 1)] = raw[((size_t)k * g->ny + j) * g->nx + i];
    cudaArray_t arr = nullptr;
    cudaTextureObject_t tex = 0;
    const cudaChannelFormatDesc cd = cudaCreateChannelDesc<float>();
    cudaError_t e = cudaMalloc3DArray(&arr, &cd, make_cudaExtent(px, py, pz));
    if (e == cudaSuccess) {
        cudaMemcpy3DParms cp;
        memset(&cp, 0, sizeof cp);
        cp.srcPtr = make_cudaPitchedPtr(pad.data(), px * sizeof(float), px, py);
        cp.dstArray = arr;
        cp.extent = make_cudaExtent(px, py, pz);
        cp.kind = cudaMemcpyHostToDevice;
        e = cudaMemcpy3D(&cp);
    }
    if (e == cudaSuccess) {
        cudaResourceDesc rd;
        memset(&rd, 0, sizeof rd);
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = arr;
        cudaTextureDesc td;
        memset(&td, 0, sizeof td);
        td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeBorder;   // zero outside
        td.filterMode = cudaFilterModeLinear;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    }
    if (e == cudaSuccess) e = launch_tex_filter(tex, positions, n, out, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (tex) cudaDestroyTextureObject(tex);
    if (arr) cudaFreeArray(arr);
    if (e != cudaSuccess) return cuda_fail(e, "texture filtering");
    return NSL_OK;
}

nsl_status nsl_debug_jitter(const nsl_march* m, uint32_t frame_id, int32_t n, uint32_t* out_hash, float* out_delta,
                            nsl_stream stream) {
    g_err.clear();
    if (!m || !out_hash || !out_delta || n < 0) return fail(NSL_ERR_INVALID_ARG, "bad arguments");
    if (n == 0) return NSL_OK;
    nsl_medium med{0.0f, 1.0f, 0.0f};
    const MarchConst mc = make_const(1, 0, &med, m);
    NSL_CUDA(launch_jitter_debug(mc, frame_id, n, out_hash, out_delta, reinterpret_cast<cudaStream_t>(stream)),
             "jitter kernel launch");
    return NSL_OK;
}

}  // extern "C"
