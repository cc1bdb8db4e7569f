"""paper_2604_03748_b200 — B200-native guiding-map ray march (Neural Six-way
Lightmaps, arXiv 2604.03748, Algorithm 1).

Thin ctypes binding over the C-ABI library ``lib/libnsl.so`` declared in
``include/nsl.h``: argument marshalling only.  Every step of the path runs in
the library's CUDA kernels (csrc/*.cu, sm_100a).  PyTorch supplies device
memory, the current CUDA stream and (in ``parallel``) torch.distributed.
There is NO CPU fallback: if the library is missing or cannot be loaded the
calls raise ``NslError``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.environ.get("NSL_LIB") or os.path.join(_HERE, "lib", "libnsl.so")   # NSL_LIB: build variants
CSRC = [os.path.join(_HERE, "csrc", f) for f in ("capi.cu", "volume.cu", "setup.cu", "march.cu", "bake.cu",
                                                  "runtime.cu", "tv.cu", "microbench.cu")]
HEADERS = [os.path.join(_HERE, "csrc", "nsl_internal.cuh"), os.path.join(_HERE, "csrc", "sampler.cuh"),
           os.path.join(_ROOT, "include", "nsl.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-cudart", "static"]

LAYOUT_LINEAR_F32, LAYOUT_QUAD_F32, LAYOUT_CORNER_F16, LAYOUT_OCT_F32, LAYOUT_BRICK_OCT_F32 = 0, 1, 2, 3, 4
LAYOUT_TEX3D_F32, LAYOUT_MORTON_OCT_F32, LAYOUT_AUTO = 5, 6, 7
LAYOUT_DEFAULT = LAYOUT_AUTO
LAYOUTS = {"linear_f32": 0, "quad_f32": 1, "corner_f16": 2, "oct_f32": 3, "brick_oct_f32": 4, "tex3d_f32": 5,
           "morton_oct_f32": 6, "auto": 7}
LAYOUT_NAMES = {v: k for k, v in LAYOUTS.items()}
LIGHTS_EXPLICIT, LIGHTS_GUIDE = 0, 1
LIGHT_MARCH, LIGHT_TV = 0, 1


class NslError(RuntimeError):
    pass


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libnsl.so for sm_100a in-tree (nvcc cross-compiles without a GPU): one nvcc
    per translation unit in parallel (objects under lib/obj/), then one shared-library link."""
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    newest = max(os.path.getmtime(p) for p in CSRC + HEADERS)
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest:
        objdir = os.path.join(os.path.dirname(LIB_PATH), "obj")
        os.makedirs(objdir, exist_ok=True)
        cflags = [f for f in NVCC_FLAGS if f not in ("-shared", "-cudart", "static")]
        objs = [os.path.join(objdir, os.path.basename(c)[:-3] + ".o") for c in CSRC]

        def compile_one(src_obj):
            src, obj = src_obj
            cmd = ["nvcc", *cflags, *(["-Xptxas", "-v"] if verbose else []), "-c", "-o", obj, src]
            return subprocess.run(cmd, capture_output=True, text=True)

        with ThreadPoolExecutor(max_workers=len(CSRC)) as ex:
            results = list(ex.map(compile_one, zip(CSRC, objs)))
        for r in results:
            if verbose or r.returncode:
                print(r.stdout + r.stderr, end="")
            if r.returncode:
                raise subprocess.CalledProcessError(r.returncode, r.args)
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                               "-o", LIB_PATH, *objs])
    return LIB_PATH


# ---------------------------------------------------------------- ABI structs (include/nsl.h)
class GridDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("origin", ctypes.c_float * 3), ("voxel_width", ctypes.c_float)]


class CameraS(ctypes.Structure):
    _fields_ = [("projection", ctypes.c_int32), ("position", ctypes.c_float * 3),
                ("forward", ctypes.c_float * 3), ("up", ctypes.c_float * 3), ("extent", ctypes.c_float),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class LightS(ctypes.Structure):
    _fields_ = [("to_light", ctypes.c_float * 3), ("rgb", ctypes.c_float * 3)]


class MediumS(ctypes.Structure):
    _fields_ = [("extinction", ctypes.c_float), ("albedo", ctypes.c_float), ("hg_g", ctypes.c_float)]


class MarchS(ctypes.Structure):
    _fields_ = [("step", ctypes.c_float), ("light_step", ctypes.c_float), ("max_steps", ctypes.c_int32),
                ("depth_tau", ctypes.c_float), ("t_min", ctypes.c_float), ("opacity_form", ctypes.c_int32),
                ("jitter", ctypes.c_int32), ("seed", ctypes.c_uint64), ("guide_axis", ctypes.c_float * 3),
                ("front_identity", ctypes.c_int32), ("light_model", ctypes.c_int32)]


class FrameConstantsS(ctypes.Structure):
    _fields_ = [("inv_dx", ctypes.c_float), ("B", ctypes.c_float * 3), ("Ex", ctypes.c_float * 3),
                ("Ey", ctypes.c_float * 3), ("Dg", ctypes.c_float * 3), ("Oe", ctypes.c_float * 3),
                ("F0", ctypes.c_float * 3), ("fwd", ctypes.c_float * 3), ("Ln", (ctypes.c_float * 3) * 4),
                ("Lg", (ctypes.c_float * 3) * 4), ("P", ctypes.c_float * 4), ("front_identity_ok", ctypes.c_int32)]


EXPORTS = ["nsl_last_error", "nsl_version", "nsl_volume_bytes", "nsl_volume_upload", "nsl_volume_check",
           "nsl_volume_release", "nsl_guiding_map", "nsl_guiding_map_batch", "nsl_guiding_map_batch_counted",
           "nsl_plan_create", "nsl_plan_execute", "nsl_plan_destroy",
           "nsl_guiding_map_host", "nsl_debug_frame_constants", "nsl_debug_jitter",
           "nsl_sixway_bake", "nsl_debug_bake_lights", "nsl_relight", "nsl_guide_lights",
           "nsl_guiding_map_animated", "nsl_bench_l1_gather", "nsl_bench_l1_peak", "nsl_volume_rebuild",
           "nsl_guiding_map_host_f16", "nsl_layout_resolve", "nsl_debug_tex_filter",
           "nsl_volume_build_launches"]


class BakeS(ctypes.Structure):
    _fields_ = [("spp", ctypes.c_int32), ("step", ctypes.c_float), ("light_step", ctypes.c_float),
                ("max_steps", ctypes.c_int32), ("t_min", ctypes.c_float), ("seed", ctypes.c_uint64)]

_lib = None


def lib():
    """Load libnsl.so (raises NslError if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NslError(f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as e:
        raise NslError(f"cannot load {LIB_PATH}: {e}") from e
    P, vp, i32, u32 = ctypes.POINTER, ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32
    L.nsl_last_error.restype = ctypes.c_char_p
    L.nsl_version.restype = ctypes.c_char_p
    L.nsl_volume_bytes.argtypes = [P(GridDesc), i32]
    L.nsl_layout_resolve.argtypes = [P(GridDesc), i32]
    L.nsl_volume_build_launches.restype = i32
    L.nsl_volume_build_launches.argtypes = [P(GridDesc), i32]
    L.nsl_debug_tex_filter.argtypes = [P(GridDesc), vp, vp, i32, vp, vp]
    L.nsl_volume_bytes.restype = ctypes.c_size_t
    L.nsl_volume_upload.argtypes = [P(GridDesc), vp, i32, i32, vp, ctypes.c_size_t, vp, P(vp)]
    L.nsl_volume_check.argtypes = [vp, vp, P(ctypes.c_uint64)]
    L.nsl_volume_release.argtypes = [vp]
    L.nsl_volume_rebuild.argtypes = [vp, vp, i32, vp]
    L.nsl_guiding_map.argtypes = [vp, P(CameraS), P(LightS), i32, i32, P(MediumS), P(MarchS), u32,
                                  vp, vp, vp, vp]
    L.nsl_guiding_map_batch.argtypes = [P(vp), i32, P(i32), P(CameraS), P(LightS), i32, i32, P(MediumS),
                                        P(MarchS), P(u32), i32, vp, vp, vp, vp]
    L.nsl_guiding_map_batch_counted.argtypes = [P(vp), i32, P(i32), P(CameraS), P(LightS), i32, i32, P(MediumS),
                                                P(MarchS), P(u32), i32, vp, vp, vp, vp]
    L.nsl_plan_create.argtypes = [P(vp), i32, P(i32), P(CameraS), P(LightS), i32, i32, P(MediumS), P(MarchS),
                                  P(u32), i32, vp, P(vp)]
    L.nsl_plan_execute.argtypes = [vp, vp, vp, vp, vp, vp]
    L.nsl_plan_destroy.argtypes = [vp]
    L.nsl_guiding_map_host.argtypes = [P(GridDesc), vp, i32, P(CameraS), P(LightS), i32, i32, P(MediumS),
                                       P(MarchS), P(u32), i32, vp, vp, vp]
    L.nsl_guiding_map_host_f16.argtypes = L.nsl_guiding_map_host.argtypes
    L.nsl_guiding_map_animated.argtypes = [P(GridDesc), P(vp), i32, P(vp), ctypes.c_size_t, P(CameraS), P(LightS),
                                           i32, i32, P(MediumS), P(MarchS), P(u32), i32, i32, vp, vp,
                                           P(ctypes.c_uint64), vp]
    L.nsl_bench_l1_gather.argtypes = [vp, i32, i32, vp, ctypes.c_size_t, P(ctypes.c_uint64), vp]
    L.nsl_bench_l1_peak.argtypes = [vp, ctypes.c_size_t, vp, i32, ctypes.c_int64, ctypes.c_int64, i32, i32, vp,
                                    ctypes.c_size_t, P(ctypes.c_uint64), vp]
    L.nsl_debug_frame_constants.argtypes = [P(GridDesc), P(CameraS), P(LightS), i32, i32, P(MediumS),
                                            P(MarchS), P(FrameConstantsS), vp]
    L.nsl_debug_jitter.argtypes = [P(MarchS), u32, i32, vp, vp, vp]
    L.nsl_sixway_bake.argtypes = [P(vp), i32, P(i32), P(CameraS), P(MediumS), P(BakeS), P(u32), i32, vp, vp, vp]
    L.nsl_debug_bake_lights.argtypes = [P(GridDesc), P(CameraS), vp, vp, vp]
    L.nsl_guide_lights.argtypes = [P(CameraS), vp, vp, P(LightS), vp]
    L.nsl_relight.argtypes = [P(CameraS), i32, vp, vp, P(LightS), i32, P(ctypes.c_float), P(ctypes.c_float),
                              vp, vp, ctypes.c_float, vp, vp]
    for name in EXPORTS[2:]:
        if name != "nsl_volume_bytes":
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def version() -> str:
    return lib().nsl_version().decode()


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().nsl_last_error().decode()
        raise NslError(f"{what} failed (status {rc}): {msg}")


# ---------------------------------------------------------------- marshalling
def _f3(v):
    return (ctypes.c_float * 3)(*[float(x) for x in v])


def grid_desc(g) -> GridDesc:
    return GridDesc(g.nx, g.ny, g.nz, _f3(g.origin), g.voxel_width)


def camera_s(c) -> CameraS:
    return CameraS(c.projection, _f3(c.position), _f3(c.forward), _f3(c.up), c.extent, c.width, c.height)


def lights_s(rows) -> ctypes.Array:
    """rows: list (frames) of lists (lights) of objects with to_light/rgb -> flat LightS array."""
    flat = [l for row in rows for l in row]
    arr = (LightS * len(flat))()
    for i, l in enumerate(flat):
        arr[i].to_light = _f3(l.to_light)
        arr[i].rgb = _f3(l.rgb)
    return arr


def medium_s(m) -> MediumS:
    return MediumS(m.extinction, m.albedo, m.hg_g)


def march_s(m) -> MarchS:
    return MarchS(m.step, m.light_step, m.max_steps, m.depth_tau, m.t_min, m.opacity_form, m.jitter,
                  m.seed & 0xFFFFFFFFFFFFFFFF, _f3(m.guide_axis), getattr(m, "front_identity", 1),
                  getattr(m, "light_model", 0))


def _stream_handle(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def layout_resolve(grid, layout: int = LAYOUT_DEFAULT) -> int:
    """The concrete layout `layout` stands for on `grid` (nsl_layout_resolve: AUTO by size)."""
    r = lib().nsl_layout_resolve(ctypes.byref(grid_desc(grid)), layout)
    if r < 0:
        raise NslError("nsl_layout_resolve: invalid grid")
    return r


def volume_build_launches(grid, layout: int = LAYOUT_DEFAULT) -> int:
    """Kernel launches of one volume build (nsl_volume_build_launches: 3 for the staged OCT
    build, else 2)."""
    n = lib().nsl_volume_build_launches(ctypes.byref(grid_desc(grid)), layout)
    if n < 0:
        raise NslError("nsl_volume_build_launches: invalid grid/layout")
    return n


def volume_bytes(grid, layout: int = LAYOUT_DEFAULT) -> int:
    n = lib().nsl_volume_bytes(ctypes.byref(grid_desc(grid)), layout)
    if n == 0:
        raise NslError("nsl_volume_bytes: invalid grid/layout")
    return n


class Volume:
    """A device volume in a sampler layout (row a1).  Owns its storage tensor."""

    def __init__(self, grid, density, layout: int = LAYOUT_DEFAULT, stream=None, storage=None):
        import torch
        self.grid = grid
        self.layout = layout_resolve(grid, layout)
        nbytes = volume_bytes(grid, layout)
        if storage is None:
            storage = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        assert storage.numel() >= nbytes and storage.is_cuda
        self.storage = storage
        self._density = density                       # keep the source alive until the copy is done
        on_dev = 1 if (hasattr(density, "is_cuda") and density.is_cuda) else 0
        if hasattr(density, "data_ptr"):
            assert density.dtype == torch.float32 and density.is_contiguous()
            ptr = density.data_ptr()
        else:
            import numpy as np
            assert density.dtype == np.float32 and density.flags["C_CONTIGUOUS"]
            ptr = density.ctypes.data
        h = ctypes.c_void_p()
        _check(lib().nsl_volume_upload(ctypes.byref(grid_desc(grid)), ptr, on_dev, layout,
                                       storage.data_ptr(), storage.numel(), _stream_handle(stream),
                                       ctypes.byref(h)), "nsl_volume_upload")
        self.handle = h

    def rebuild(self, density, stream=None):
        """Rebuild this volume's layout in place from new density values (nsl_volume_rebuild):
        same grid, layout, storage (and TEX3D array); plans referencing it see the new values."""
        import torch
        on_dev = 1 if (hasattr(density, "is_cuda") and density.is_cuda) else 0
        if hasattr(density, "data_ptr"):
            assert density.dtype == torch.float32 and density.is_contiguous()
            ptr = density.data_ptr()
        else:
            import numpy as np
            assert density.dtype == np.float32 and density.flags["C_CONTIGUOUS"]
            ptr = density.ctypes.data
        self._density = density
        _check(lib().nsl_volume_rebuild(self.handle, ptr, on_dev, _stream_handle(stream)), "nsl_volume_rebuild")
        return self

    def check(self, stream=None) -> int:
        n = ctypes.c_uint64()
        _check(lib().nsl_volume_check(self.handle, _stream_handle(stream), ctypes.byref(n)), "nsl_volume_check")
        return n.value

    def release(self):
        if getattr(self, "handle", None) is not None and _lib is not None:
            _lib.nsl_volume_release(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def guiding_map(vol: Volume, cam, lights, light_mode, medium, march, frame_id: int, out_rgbt, out_depth,
                out_debug=None, stream=None):
    """One frame (rows a2-a8).  out_rgbt: cuda float32 [H,W,4]; out_depth [H,W]; out_debug [H,W,6] int32 or None."""
    ls = lights_s([lights])
    _check(lib().nsl_guiding_map(vol.handle, ctypes.byref(camera_s(cam)), ls, len(lights), light_mode,
                                 ctypes.byref(medium_s(medium)), ctypes.byref(march_s(march)), frame_id,
                                 _ptr(out_rgbt), _ptr(out_depth), _ptr(out_debug), _stream_handle(stream)),
           "nsl_guiding_map")


def guiding_map_batch(vols: Sequence[Volume], frame_vol: Sequence[int], cams, lights, light_mode, medium, march,
                      frame_ids: Sequence[int], out_rgbt, out_depth, out_debug=None, stream=None):
    """F frames in one launch (row a9).  lights: F rows of n_lights.  Outputs [F,H,W,4], [F,H,W], [F,H,W,6]."""
    F = len(cams)
    n_l = len(lights[0])
    hv = (ctypes.c_void_p * len(vols))(*[v.handle.value for v in vols])
    fv = (ctypes.c_int32 * F)(*frame_vol)
    cs = (CameraS * F)(*[camera_s(c) for c in cams])
    fid = (ctypes.c_uint32 * F)(*[int(x) & 0xFFFFFFFF for x in frame_ids])
    _check(lib().nsl_guiding_map_batch(hv, len(vols), fv, cs, lights_s(lights), n_l, light_mode,
                                       ctypes.byref(medium_s(medium)), ctypes.byref(march_s(march)), fid, F,
                                       _ptr(out_rgbt), _ptr(out_depth), _ptr(out_debug), _stream_handle(stream)),
           "nsl_guiding_map_batch")


def guiding_map_batch_counted(vols, frame_vol, cams, lights, light_mode, medium, march, frame_ids, out_rgbt,
                              out_depth, stream=None) -> dict:
    """The timed fast path plus work counters: returns canonical primary/light
    sample counts, trilinear gathers actually executed and occupied samples."""
    import torch
    F = len(cams)
    counters = torch.zeros(8, dtype=torch.int64, device="cuda")
    hv = (ctypes.c_void_p * len(vols))(*[v.handle.value for v in vols])
    fv = (ctypes.c_int32 * F)(*frame_vol)
    cs = (CameraS * F)(*[camera_s(c) for c in cams])
    fid = (ctypes.c_uint32 * F)(*[int(x) & 0xFFFFFFFF for x in frame_ids])
    _check(lib().nsl_guiding_map_batch_counted(hv, len(vols), fv, cs, lights_s(lights), len(lights[0]), light_mode,
                                               ctypes.byref(medium_s(medium)), ctypes.byref(march_s(march)), fid, F,
                                               _ptr(out_rgbt), _ptr(out_depth), counters.data_ptr(),
                                               _stream_handle(stream)), "nsl_guiding_map_batch_counted")
    c = counters.cpu().tolist()
    return {"primary_samples": c[0], "light_samples": c[1], "gathers": c[2], "occupied_samples": c[3],
            "tested_primary": c[4], "tested_light": c[5], "canonical_samples": c[0] + c[1]}


class Plan:
    """A prepared batch (nsl_plan_*): per-frame inputs marshalled and uploaded once;
    execute() enqueues only the setup and march kernels (no host work per call)."""

    def __init__(self, vols, frame_vol, cams, lights, light_mode, medium, march, frame_ids, stream=None):
        F = len(cams)
        self.F, self.H, self.W = F, cams[0].height, cams[0].width
        hv = (ctypes.c_void_p * len(vols))(*[v.handle.value for v in vols])
        fv = (ctypes.c_int32 * F)(*frame_vol)
        cs = (CameraS * F)(*[camera_s(c) for c in cams])
        fid = (ctypes.c_uint32 * F)(*[int(x) & 0xFFFFFFFF for x in frame_ids])
        self._vols = list(vols)      # the plan holds raw storage pointers: keep the storage alive
        h = ctypes.c_void_p()
        _check(lib().nsl_plan_create(hv, len(vols), fv, cs, lights_s(lights), len(lights[0]), light_mode,
                                     ctypes.byref(medium_s(medium)), ctypes.byref(march_s(march)), fid, F,
                                     _stream_handle(stream), ctypes.byref(h)), "nsl_plan_create")
        self.handle = h

    def execute(self, out_rgbt, out_depth, out_debug=None, counters=None, stream=None):
        _check(lib().nsl_plan_execute(self.handle, _ptr(out_rgbt), _ptr(out_depth), _ptr(out_debug), _ptr(counters),
                                      _stream_handle(stream)), "nsl_plan_execute")

    def execute_counted(self, out_rgbt, out_depth, stream=None) -> dict:
        import torch
        c = torch.zeros(8, dtype=torch.int64, device="cuda")
        self.execute(out_rgbt, out_depth, None, c, stream)
        c = c.cpu().tolist()
        return {"primary_samples": c[0], "light_samples": c[1], "gathers": c[2], "occupied_samples": c[3],
                "tested_primary": c[4], "tested_light": c[5], "canonical_samples": c[0] + c[1]}

    def destroy(self):
        if getattr(self, "handle", None) is not None and _lib is not None:
            _lib.nsl_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def make_plan(w, vols, march=None, stream=None) -> Plan:
    return Plan(vols, w.frame_vol, w.cameras, w.lights, w.light_mode, w.medium, march or w.march, w.frame_ids,
                stream=stream)


def bake_s(b) -> BakeS:
    return BakeS(b.spp, b.step, b.light_step, b.max_steps, b.t_min, b.seed & 0xFFFFFFFFFFFFFFFF)


def sixway_bake(vols, frame_vol, cams, medium, bake, frame_ids, out, counters=None, stream=None):
    """NEXT-1 six-way bake.  out: cuda float32 [F, H, W, 2, 4] in the Fig. 2
    packing (right, top, back, T)(left, bottom, front, E); counters: int64[1] (gathers) or None."""
    F = len(cams)
    hv = (ctypes.c_void_p * len(vols))(*[v.handle.value for v in vols])
    fv = (ctypes.c_int32 * F)(*frame_vol)
    cs = (CameraS * F)(*[camera_s(c) for c in cams])
    fid = (ctypes.c_uint32 * F)(*[int(x) & 0xFFFFFFFF for x in frame_ids])
    _check(lib().nsl_sixway_bake(hv, len(vols), fv, cs, ctypes.byref(medium_s(medium)), ctypes.byref(bake_s(bake)),
                                 fid, F, _ptr(out), _ptr(counters), _stream_handle(stream)), "nsl_sixway_bake")


def debug_bake_lights(grid, cam, stream=None):
    import numpy as np
    Lg = np.zeros((6, 3), np.float32)
    Ln = np.zeros((6, 3), np.float32)
    _check(lib().nsl_debug_bake_lights(ctypes.byref(grid_desc(grid)), ctypes.byref(camera_s(cam)), Lg.ctypes.data,
                                       Ln.ctypes.data, _stream_handle(stream)), "nsl_debug_bake_lights")
    return Lg, Ln


def relight(cams, maps, lights, out, depth=None, bg=(0.0, 0.0, 0.0), emis=(0.0, 0.0, 0.0), shadow_cams=None,
            shadow_maps=None, bias: float = 2e-3, stream=None):
    """NEXT-2/3 relight + composite + depth shadow.  maps: cuda float32 [F,H,W,2,4]
    (Fig. 2 packing); depth: cuda [F,H,W] or None; lights: F rows of n lights; shadow_cams /
    shadow_maps: F rows of n entries (Camera / cuda float32 [Hs,Ws] or None).  out: cuda [F,H,W,4]."""
    RelightCall(cams, maps, lights, out, depth, bg, emis, shadow_cams, shadow_maps, bias)(stream)


class RelightCall:
    """nsl_relight with its arguments marshalled once (for repeated launches on the same
    buffers, e.g. per-frame relighting of a resident batch); ``call(stream)`` launches."""

    def __init__(self, cams, maps, lights, out, depth=None, bg=(0.0, 0.0, 0.0), emis=(0.0, 0.0, 0.0),
                 shadow_cams=None, shadow_maps=None, bias: float = 2e-3):
        F = len(cams)
        n = len(lights[0])
        f3 = ctypes.c_float * 3
        self._keep = [maps, depth, out, shadow_maps]
        self.cs = (CameraS * F)(*[camera_s(c) for c in cams])
        self.ls = lights_s(lights)
        self.bg, self.emis = f3(*bg), f3(*emis)
        self.sc = self.sm = None
        if shadow_maps is not None:
            self.sc = (CameraS * (F * n))(*[camera_s(c) if c is not None else CameraS()
                                            for row in shadow_cams for c in row])
            self.sm = (ctypes.c_void_p * (F * n))(*[None if t is None else t.data_ptr()
                                                    for row in shadow_maps for t in row])
        self.args = (self.cs, F, _ptr(maps), _ptr(depth), self.ls, n, self.bg, self.emis,
                     None if self.sc is None else ctypes.addressof(self.sc),
                     None if self.sm is None else ctypes.addressof(self.sm), bias, _ptr(out))

    def __call__(self, stream=None):
        _check(lib().nsl_relight(*self.args, _stream_handle(stream)), "nsl_relight")


def guide_lights(cam, axis=None, rgb=None, stream=None):
    """The surrogate light set of eq:approx (front, top, bottom) for a camera, as the device
    computes it: a list of three (to_light, rgb) tuples."""
    out = (LightS * 3)()
    ax = None if axis is None else _f3(axis)
    col = None if rgb is None else _f3(rgb)
    _check(lib().nsl_guide_lights(ctypes.byref(camera_s(cam)), None if ax is None else ctypes.addressof(ax),
                                  None if col is None else ctypes.addressof(col), out, _stream_handle(stream)),
           "nsl_guide_lights")
    return [(tuple(out[l].to_light), tuple(out[l].rgb)) for l in range(3)]


def run_bake(w, bake, layout: int = LAYOUT_DEFAULT, vols=None, out=None, stream=None):
    """Six-way bake of every frame of an nsl_inputs.Workload; returns the [F, H, W, 2, 4] tensor."""
    import torch
    if vols is None:
        vols = upload_workload_volumes(w, layout, stream=stream)
    if out is None:
        out = torch.empty((w.n_frames, w.height, w.width, 2, 4), dtype=torch.float32, device="cuda")
    sixway_bake(vols, w.frame_vol, w.cameras, w.medium, bake, w.frame_ids, out, stream=stream)
    return out


def guiding_map_host(grid, host_density, layout, cams, lights, light_mode, medium, march, frame_ids,
                     host_rgbt, host_depth, stream=None):
    """End-to-end with HOST buffers (torch CPU tensors, pinned for async DMA): upload + layout + march + download."""
    F = len(cams)
    cs = (CameraS * F)(*[camera_s(c) for c in cams])
    fid = (ctypes.c_uint32 * F)(*[int(x) & 0xFFFFFFFF for x in frame_ids])
    _check(lib().nsl_guiding_map_host(ctypes.byref(grid_desc(grid)), host_density.data_ptr(), layout, cs,
                                      lights_s(lights), len(lights[0]), light_mode, ctypes.byref(medium_s(medium)),
                                      ctypes.byref(march_s(march)), fid, F, host_rgbt.data_ptr(),
                                      host_depth.data_ptr(), _stream_handle(stream)), "nsl_guiding_map_host")


def guiding_map_host_f16(grid, host_density, layout, cams, lights, light_mode, medium, march, frame_ids,
                         host_rgbt_h, host_depth_h, stream=None):
    """guiding_map_host with the compact download (nsl_guiding_map_host_f16): host_rgbt_h /
    host_depth_h are torch.float16 CPU tensors [F,H,W,4] / [F,H,W] (the fp32 maps rounded RNE)."""
    import torch
    assert host_rgbt_h.dtype == torch.float16 and host_depth_h.dtype == torch.float16
    F = len(cams)
    cs = (CameraS * F)(*[camera_s(c) for c in cams])
    fid = (ctypes.c_uint32 * F)(*[int(x) & 0xFFFFFFFF for x in frame_ids])
    _check(lib().nsl_guiding_map_host_f16(ctypes.byref(grid_desc(grid)), host_density.data_ptr(), layout, cs,
                                          lights_s(lights), len(lights[0]), light_mode,
                                          ctypes.byref(medium_s(medium)), ctypes.byref(march_s(march)), fid, F,
                                          host_rgbt_h.data_ptr(), host_depth_h.data_ptr(), _stream_handle(stream)),
           "nsl_guiding_map_host_f16")


class Animated:
    """nsl_guiding_map_animated (rows a1 + a9, C4) with the host arguments marshalled once:
    frame f's device density densities[f] is laid out into storages[f] and marched with
    cams[f]; the layouts of the next chunk of frames build on a side stream while the current
    chunk marches.  Calling it re-runs the whole step (e.g. after the simulator refreshed the
    densities in place)."""

    def __init__(self, grid, densities, layout, storages, cams, lights, light_mode, medium, march, frame_ids,
                 chunk: int = 0):
        F = len(cams)
        assert len(densities) == F and len(storages) == F
        for d in densities:
            assert d.is_cuda and d.is_contiguous()
        self._keep = (list(densities), list(storages))
        self.F, self.layout, self.chunk, self.n_l, self.light_mode = F, layout, chunk, len(lights[0]), light_mode
        self.nbytes = min(t.numel() for t in storages)
        self.g = grid_desc(grid)
        self.dp = (ctypes.c_void_p * F)(*[d.data_ptr() for d in densities])
        self.sp = (ctypes.c_void_p * F)(*[t.data_ptr() for t in storages])
        self.cs = (CameraS * F)(*[camera_s(c) for c in cams])
        self.ls = lights_s(lights)
        self.med, self.mar = medium_s(medium), march_s(march)
        self.fid = (ctypes.c_uint32 * F)(*[int(x) & 0xFFFFFFFF for x in frame_ids])

    def __call__(self, out_rgbt, out_depth, check: bool = False, stream=None) -> Optional[int]:
        """check=True synchronises and returns the number of invalid density values over all frames."""
        n = ctypes.c_uint64()
        _check(lib().nsl_guiding_map_animated(ctypes.byref(self.g), self.dp, self.layout, self.sp, self.nbytes,
                                              self.cs, self.ls, self.n_l, self.light_mode, ctypes.byref(self.med),
                                              ctypes.byref(self.mar), self.fid, self.F, self.chunk,
                                              _ptr(out_rgbt), _ptr(out_depth), ctypes.byref(n) if check else None,
                                              _stream_handle(stream)), "nsl_guiding_map_animated")
        return n.value if check else None


def guiding_map_animated(grid, densities, layout, storages, cams, lights, light_mode, medium, march, frame_ids,
                         out_rgbt, out_depth, chunk: int = 0, check: bool = False, stream=None) -> Optional[int]:
    """One-shot form of Animated (marshals the host arguments on every call)."""
    return Animated(grid, densities, layout, storages, cams, lights, light_mode, medium, march, frame_ids,
                    chunk)(out_rgbt, out_depth, check=check, stream=stream)


def bench_l1_gather(vol: Volume, sink, waves: int = 4, reps: int = 64, stream=None) -> int:
    """Enqueue the sampler microbenchmark on `vol` (nsl_bench_l1_gather); returns the samples it takes."""
    n = ctypes.c_uint64()
    _check(lib().nsl_bench_l1_gather(vol.handle, waves, reps, sink.data_ptr(), sink.numel(), ctypes.byref(n),
                                     _stream_handle(stream)), "nsl_bench_l1_gather")
    return n.value


def bench_l1_peak(buf, lane_off, stride: int = 0, span: int = 1, waves: int = 4, reps: int = 64, sink=None,
                  stream=None) -> int:
    """Enqueue the hardware L1/TEX gather ceiling (nsl_bench_l1_peak); returns the lane bytes it loads.
    buf: cuda float32 (32-B aligned); lane_off: cuda int32 [16, 32] element offsets."""
    n = ctypes.c_uint64()
    max_off = int(lane_off.max().item())
    _check(lib().nsl_bench_l1_peak(buf.data_ptr(), buf.numel(), lane_off.data_ptr(), max_off, stride, span, waves,
                                   reps, sink.data_ptr(), sink.numel(), ctypes.byref(n), _stream_handle(stream)),
           "nsl_bench_l1_peak")
    return n.value


def debug_tex_filter(grid, density, positions, stream=None):
    """Hardware trilinear (texture) filtering of `density` (cuda float32 [nz,ny,nx]) at padded-index
    positions (cuda float32 [n,3]) -> cuda float32 [n] (nsl_debug_tex_filter)."""
    import torch
    out = torch.empty(positions.shape[0], dtype=torch.float32, device="cuda")
    _check(lib().nsl_debug_tex_filter(ctypes.byref(grid_desc(grid)), density.data_ptr(), positions.data_ptr(),
                                      positions.shape[0], out.data_ptr(), _stream_handle(stream)),
           "nsl_debug_tex_filter")
    return out


def debug_frame_constants(grid, cam, lights, light_mode, medium, march, stream=None) -> dict:
    import numpy as np
    out = FrameConstantsS()
    _check(lib().nsl_debug_frame_constants(ctypes.byref(grid_desc(grid)), ctypes.byref(camera_s(cam)),
                                           lights_s([lights]), len(lights), light_mode,
                                           ctypes.byref(medium_s(medium)), ctypes.byref(march_s(march)),
                                           ctypes.byref(out), _stream_handle(stream)), "nsl_debug_frame_constants")
    n = len(lights)
    return {"inv_dx": np.float32(out.inv_dx),
            "B": np.array(out.B, np.float32), "Ex": np.array(out.Ex, np.float32),
            "Ey": np.array(out.Ey, np.float32), "Dg": np.array(out.Dg, np.float32),
            "Oe": np.array(out.Oe, np.float32), "F0": np.array(out.F0, np.float32),
            "fwd": np.array(out.fwd, np.float32),
            "Ln": np.array([list(out.Ln[i]) for i in range(n)], np.float32),
            "Lg": np.array([list(out.Lg[i]) for i in range(n)], np.float32),
            "P": np.array(list(out.P)[:n], np.float32), "front_identity_ok": out.front_identity_ok}


def debug_jitter(march, frame_id: int, out_hash, out_delta, stream=None):
    _check(lib().nsl_debug_jitter(ctypes.byref(march_s(march)), frame_id, out_hash.numel(), out_hash.data_ptr(),
                                  out_delta.data_ptr(), _stream_handle(stream)), "nsl_debug_jitter")


# ---------------------------------------------------------------- workload driver (marshalling only)
def upload_workload_volumes(w, layout: int = LAYOUT_DEFAULT, vol_indices=None, stream=None) -> List[Volume]:
    """Upload the workload's distinct volumes (host -> device layout kernel)."""
    import torch
    idx = range(len(w.volume_specs)) if vol_indices is None else vol_indices
    vols = []
    for i in idx:
        d = torch.from_numpy(w.volume(i)).cuda(non_blocking=False)
        vols.append(Volume(w.grid, d, layout, stream=stream))
    return vols


def alloc_outputs(F: int, H: int, W: int, debug: bool = False):
    import torch
    rgbt = torch.empty((F, H, W, 4), dtype=torch.float32, device="cuda")
    depth = torch.empty((F, H, W), dtype=torch.float32, device="cuda")
    dbg = torch.empty((F, H, W, 6), dtype=torch.int32, device="cuda") if debug else None
    return rgbt, depth, dbg


def run_workload(w, layout: int = LAYOUT_DEFAULT, debug: bool = False, vols=None, outputs=None, march=None,
                 stream=None):
    """March every frame of an nsl_inputs.Workload in one batched call; returns (rgbt, depth, debug)."""
    if vols is None:
        vols = upload_workload_volumes(w, layout, stream=stream)
    if outputs is None:
        outputs = alloc_outputs(w.n_frames, w.height, w.width, debug)
    rgbt, depth, dbg = outputs
    guiding_map_batch(vols, w.frame_vol, w.cameras, w.lights, w.light_mode, w.medium, march or w.march,
                      w.frame_ids, rgbt, depth, dbg, stream=stream)
    return rgbt, depth, dbg
