"""CPU oracle of the guiding-map ray march — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product (``paper_2604_03748_b200``) never imports it, and it never imports
the product: the two share no code (DESIGN.md §3 "Oracle independence").

The arithmetic lives in ``nsl_oracle.c`` (plain single-threaded C, fp64
values, prescribed fp32 index ops, built with ``-ffp-contract=off``), written
from DESIGN.md §2, which restates PAPER.md Algorithm 1 (L394-407), eq:approx
(L361-365) and §4.2 (L410).  This module is ctypes marshalling only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nsl_oracle.c")
_HDR = os.path.join(_HERE, "nsl_oracle.h")
LIB_PATH = os.path.join(_HERE, "libnsl_oracle.so")
CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
          "-D_GNU_SOURCE"]
_lib = None


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest:
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB_PATH, _SRC, "-lm"])
    return LIB_PATH


class OrcGrid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("origin", ctypes.c_float * 3), ("voxel_width", ctypes.c_float)]


class OrcCamera(ctypes.Structure):
    _fields_ = [("projection", ctypes.c_int32), ("position", ctypes.c_float * 3),
                ("forward", ctypes.c_float * 3), ("up", ctypes.c_float * 3),
                ("extent", ctypes.c_float), ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class OrcLight(ctypes.Structure):
    _fields_ = [("to_light", ctypes.c_float * 3), ("rgb", ctypes.c_float * 3)]


class OrcMedium(ctypes.Structure):
    _fields_ = [("extinction", ctypes.c_float), ("albedo", ctypes.c_float), ("hg_g", ctypes.c_float)]


class OrcMarch(ctypes.Structure):
    _fields_ = [("step", ctypes.c_float), ("light_step", ctypes.c_float),
                ("max_steps", ctypes.c_int32), ("depth_tau", ctypes.c_float),
                ("t_min", ctypes.c_float), ("opacity_form", ctypes.c_int32),
                ("jitter", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("guide_axis", ctypes.c_float * 3), ("light_model", ctypes.c_int32)]


class OrcFrameConstants(ctypes.Structure):
    _fields_ = [("inv_dx", ctypes.c_float), ("B", ctypes.c_float * 3), ("Ex", ctypes.c_float * 3),
                ("Ey", ctypes.c_float * 3), ("Dg", ctypes.c_float * 3), ("Oe", ctypes.c_float * 3),
                ("F0", ctypes.c_float * 3), ("fwd", ctypes.c_float * 3),
                ("Ln", (ctypes.c_float * 3) * 4), ("Lg", (ctypes.c_float * 3) * 4),
                ("P", ctypes.c_float * 4), ("P64", ctypes.c_double * 4)]


DENSITY_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.POINTER(ctypes.c_float), ctypes.c_void_p)


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        lib.orc_hg.argtypes = [ctypes.c_double, ctypes.c_double]
        lib.orc_hg.restype = ctypes.c_double
        lib.orc_fmix32.argtypes = [ctypes.c_uint32]
        lib.orc_fmix32.restype = ctypes.c_uint32
        lib.orc_jitter_hash.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32]
        lib.orc_jitter_hash.restype = ctypes.c_uint32
        lib.orc_jitter_delta.argtypes = [P(OrcMarch), ctypes.c_uint32, ctypes.c_uint32]
        lib.orc_jitter_delta.restype = ctypes.c_float
        lib.orc_sample.argtypes = [P(OrcGrid), ctypes.c_void_p, P(ctypes.c_float)]
        lib.orc_sample.restype = ctypes.c_double
        lib.orc_frame_constants_compute.argtypes = [P(OrcGrid), P(OrcCamera), P(OrcLight), ctypes.c_int32,
                                                    ctypes.c_int32, P(OrcMedium), P(OrcMarch),
                                                    P(OrcFrameConstants)]
        lib.orc_frame_constants_compute.restype = ctypes.c_int
        lib.orc_guiding_map.argtypes = [P(OrcGrid), ctypes.c_void_p, DENSITY_FN, ctypes.c_void_p,
                                        P(OrcCamera), P(OrcLight), ctypes.c_int32, ctypes.c_int32,
                                        P(OrcMedium), P(OrcMarch), ctypes.c_uint32, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int32]
        lib.orc_guiding_map.restype = ctypes.c_int
        _lib = lib
    return _lib


# ------------------------------------------------------------------ marshalling
def _grid(g) -> OrcGrid:
    return OrcGrid(g.nx, g.ny, g.nz, (ctypes.c_float * 3)(*g.origin), g.voxel_width)


def _camera(c) -> OrcCamera:
    f3 = ctypes.c_float * 3
    return OrcCamera(c.projection, f3(*c.position), f3(*c.forward), f3(*c.up), c.extent, c.width, c.height)


def _lights(ls):
    arr = (OrcLight * max(1, len(ls)))()
    for i, l in enumerate(ls):
        arr[i].to_light = (ctypes.c_float * 3)(*l.to_light)
        arr[i].rgb = (ctypes.c_float * 3)(*l.rgb)
    return arr


def _medium(m) -> OrcMedium:
    return OrcMedium(m.extinction, m.albedo, m.hg_g)


def _march(m) -> OrcMarch:
    return OrcMarch(m.step, m.light_step, m.max_steps, m.depth_tau, m.t_min, m.opacity_form,
                    m.jitter, m.seed & 0xFFFFFFFFFFFFFFFF, (ctypes.c_float * 3)(*m.guide_axis),
                    getattr(m, "light_model", 0))


def hg(g: float, cos_theta: float) -> float:
    return _load().orc_hg(g, cos_theta)


def fmix32(h: int) -> int:
    return _load().orc_fmix32(h & 0xFFFFFFFF)


def jitter_hash(seed: int, frame_id: int, pixel: int) -> int:
    return _load().orc_jitter_hash(seed & 0xFFFFFFFFFFFFFFFF, frame_id, pixel)


def jitter_delta(march, frame_id: int, pixel: int) -> float:
    m = _march(march)
    return _load().orc_jitter_delta(ctypes.byref(m), frame_id, pixel)


def sample(grid, vals: np.ndarray, u) -> float:
    v = np.ascontiguousarray(vals, dtype=np.float32)
    g = _grid(grid)
    uu = (ctypes.c_float * 3)(*u)
    return _load().orc_sample(ctypes.byref(g), v.ctypes.data, uu)


def frame_constants(grid, cam, lights, light_mode, medium, march) -> dict:
    out = OrcFrameConstants()
    ls = _lights(lights)
    rc = _load().orc_frame_constants_compute(ctypes.byref(_grid(grid)), ctypes.byref(_camera(cam)), ls,
                                             len(lights), light_mode, ctypes.byref(_medium(medium)),
                                             ctypes.byref(_march(march)), ctypes.byref(out))
    if rc:
        raise ValueError("orc_frame_constants_compute rejected its arguments")
    n = len(lights)
    return {
        "inv_dx": np.float32(out.inv_dx),
        "B": np.array(out.B, np.float32), "Ex": np.array(out.Ex, np.float32),
        "Ey": np.array(out.Ey, np.float32), "Dg": np.array(out.Dg, np.float32),
        "Oe": np.array(out.Oe, np.float32), "F0": np.array(out.F0, np.float32),
        "fwd": np.array(out.fwd, np.float32),
        "Ln": np.array([list(out.Ln[i]) for i in range(n)], np.float32),
        "Lg": np.array([list(out.Lg[i]) for i in range(n)], np.float32),
        "P": np.array(list(out.P)[:n], np.float32),
        "P64": np.array(list(out.P64)[:n], np.float64),
    }


def guiding_map(grid, vals: Optional[np.ndarray], cam, lights, light_mode, medium, march,
                frame_id: int = 0, pixels: Optional[Sequence[int]] = None, density_fn=None,
                forced_hit=None, forced_term=None, no_clip_n: int = 0) -> dict:
    """Run the oracle on one frame.  Returns rgbt (n,4) f64, depth (n,) f32,
    debug (n,6) u32, margin (n,2) f64, and the pixel list used."""
    lib = _load()
    W, H = cam.width, cam.height
    if pixels is None:
        pix = None
        n = W * H
    else:
        pix = np.ascontiguousarray(np.asarray(pixels, dtype=np.int64))
        n = int(pix.size)
    rgbt = np.zeros((n, 4), np.float64)
    depth = np.zeros((n,), np.float32)
    debug = np.zeros((n, 6), np.uint32)
    margin = np.zeros((n, 2), np.float64)
    v = None
    if vals is not None:
        v = np.ascontiguousarray(vals, dtype=np.float32)
        assert v.size == grid.nx * grid.ny * grid.nz
    fh = None if forced_hit is None else np.ascontiguousarray(np.asarray(forced_hit, np.int32))
    ft = None if forced_term is None else np.ascontiguousarray(np.asarray(forced_term, np.int32))
    cb = DENSITY_FN(density_fn) if density_fn is not None else DENSITY_FN()
    ls = _lights(lights)
    rc = lib.orc_guiding_map(ctypes.byref(_grid(grid)), None if v is None else v.ctypes.data, cb, None,
                             ctypes.byref(_camera(cam)), ls, len(lights), light_mode,
                             ctypes.byref(_medium(medium)), ctypes.byref(_march(march)), frame_id, n,
                             None if pix is None else pix.ctypes.data,
                             rgbt.ctypes.data, depth.ctypes.data, debug.ctypes.data, margin.ctypes.data,
                             None if fh is None else fh.ctypes.data,
                             None if ft is None else ft.ctypes.data, no_clip_n)
    if rc:
        raise ValueError("orc_guiding_map rejected its arguments")
    return {"rgbt": rgbt, "depth": depth, "debug": debug, "margin": margin,
            "pixels": np.arange(n, dtype=np.int64) if pix is None else pix}


def run_workload_frame(w, f: int, pixels=None, **kw) -> dict:
    """Oracle on frame f (local index) of an nsl_inputs.Workload."""
    return guiding_map(w.grid, w.volume(w.frame_vol[f]), w.cameras[f], w.lights[f], w.light_mode,
                       w.medium, w.march, frame_id=w.frame_ids[f], pixels=pixels, **kw)


# ------------------------------------------------------------------ NEXT-1 six-way bake
class OrcBake(ctypes.Structure):
    _fields_ = [("spp", ctypes.c_int32), ("step", ctypes.c_float), ("light_step", ctypes.c_float),
                ("max_steps", ctypes.c_int32), ("t_min", ctypes.c_float), ("seed", ctypes.c_uint64)]


def _bake_s(b) -> OrcBake:
    return OrcBake(b.spp, b.step, b.light_step, b.max_steps, b.t_min, b.seed & 0xFFFFFFFFFFFFFFFF)


def _load_bake():
    L = _load()
    if not getattr(L, "_bake_ready", False):
        P = ctypes.POINTER
        L.orc_bake_random.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                      P(ctypes.c_float)]
        L.orc_bake_light_constants.argtypes = [P(OrcGrid), P(OrcCamera), ctypes.c_void_p, ctypes.c_void_p]
        L.orc_sixway_bake.argtypes = [P(OrcGrid), ctypes.c_void_p, DENSITY_FN, ctypes.c_void_p, P(OrcCamera),
                                      P(OrcMedium), P(OrcBake), ctypes.c_uint32, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p]
        L.orc_sixway_bake.restype = ctypes.c_int
        L._bake_ready = True
    return L


def bake_random(seed: int, frame: int, pixel: int, sample: int):
    out = (ctypes.c_float * 4)()
    _load_bake().orc_bake_random(seed & 0xFFFFFFFFFFFFFFFF, frame, pixel, sample, out)
    return np.array(list(out), np.float32)


def bake_light_constants(grid, cam):
    Lg = np.zeros((6, 3), np.float32)
    Ln = np.zeros((6, 3), np.float32)
    _load_bake().orc_bake_light_constants(ctypes.byref(_grid(grid)), ctypes.byref(_camera(cam)), Lg.ctypes.data,
                                          Ln.ctypes.data)
    return Lg, Ln


def sixway_bake(grid, vals, cam, medium, bake, frame_id: int = 0, pixels=None, density_fn=None) -> dict:
    """Oracle of the six-way bake (B1-B6).  Returns out (n, 8) f64 in the Fig. 2 packing
    (right, top, back, T, left, bottom, front, E), steps (n,) u32, pixels."""
    L = _load_bake()
    W, H = cam.width, cam.height
    if pixels is None:
        pix, n = None, W * H
    else:
        pix = np.ascontiguousarray(np.asarray(pixels, dtype=np.int64))
        n = int(pix.size)
    out = np.zeros((n, 8), np.float64)
    steps = np.zeros((n,), np.uint32)
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.float32)
    cb = DENSITY_FN(density_fn) if density_fn is not None else DENSITY_FN()
    rc = L.orc_sixway_bake(ctypes.byref(_grid(grid)), None if v is None else v.ctypes.data, cb, None,
                           ctypes.byref(_camera(cam)), ctypes.byref(_medium(medium)), ctypes.byref(_bake_s(bake)),
                           frame_id, n, None if pix is None else pix.ctypes.data, out.ctypes.data,
                           steps.ctypes.data)
    if rc:
        raise ValueError("orc_sixway_bake rejected its arguments")
    return {"out": out, "steps": steps, "pixels": np.arange(n, dtype=np.int64) if pix is None else pix}


# ------------------------------------------------------------------ NEXT-2/3 relight + shadow
def _load_relight():
    L = _load_bake()
    if not getattr(L, "_relight_ready", False):
        P = ctypes.POINTER
        L.orc_relight_weights.argtypes = [P(OrcCamera), P(OrcLight), ctypes.c_int32, ctypes.c_void_p]
        L.orc_relight.argtypes = [P(OrcCamera), ctypes.c_void_p, ctypes.c_void_p, P(OrcLight), ctypes.c_int32,
                                  P(ctypes.c_float), P(ctypes.c_float), ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_float, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p]
        L.orc_relight.restype = ctypes.c_int
        L._relight_ready = True
    return L


def relight_weights(cam, lights):
    c = np.zeros((len(lights), 3), np.float32)
    _load_relight().orc_relight_weights(ctypes.byref(_camera(cam)), _lights(lights), len(lights), c.ctypes.data)
    return c


def relight(cam, maps8, lights, bg=(0.0, 0.0, 0.0), emis=(0.0, 0.0, 0.0), depth=None, shadow_cams=None,
            shadow_maps=None, bias=2e-3, pixels=None) -> dict:
    """Oracle of R1-R3.  maps8: float32 [H, W, 8] (Fig. 2 packing); depth: float32 [H, W] or None;
    shadow_cams / shadow_maps: per light (Camera, float32 [Hs, Ws] or None).  Returns out (n, 4) f64
    (r, g, b, alpha), margin (n,), pixels."""
    L = _load_relight()
    W, H = cam.width, cam.height
    m = np.ascontiguousarray(maps8, dtype=np.float32).reshape(-1)
    d = None if depth is None else np.ascontiguousarray(depth, dtype=np.float32).reshape(-1)
    pix = None if pixels is None else np.ascontiguousarray(np.asarray(pixels, np.int64))
    n = W * H if pix is None else int(pix.size)
    out = np.zeros((n, 4), np.float64)
    margin = np.zeros((n,), np.float64)
    sc_arr = None
    sm_ptrs = None
    keep = []
    if shadow_cams is not None:
        sc_arr = (OrcCamera * len(lights))(*[_camera(c) if c is not None else OrcCamera() for c in shadow_cams])
        sm_ptrs = (ctypes.c_void_p * len(lights))()
        for i, smap in enumerate(shadow_maps):
            if smap is not None:
                a = np.ascontiguousarray(smap, dtype=np.float32)
                keep.append(a)
                sm_ptrs[i] = a.ctypes.data
    f3 = ctypes.c_float * 3
    rc = L.orc_relight(ctypes.byref(_camera(cam)), m.ctypes.data, None if d is None else d.ctypes.data,
                       _lights(lights), len(lights), f3(*bg), f3(*emis),
                       None if sc_arr is None else ctypes.addressof(sc_arr),
                       None if sm_ptrs is None else ctypes.addressof(sm_ptrs), bias, n,
                       None if pix is None else pix.ctypes.data, out.ctypes.data, margin.ctypes.data)
    if rc:
        raise ValueError("orc_relight rejected its arguments")
    return {"out": out, "margin": margin, "pixels": np.arange(n, dtype=np.int64) if pix is None else pix}


# ------------------------------------------------------------------ NEXT-4 transmittance volume
class OrcTvLattice(ctypes.Structure):
    _fields_ = [("d", ctypes.c_double * 3), ("dhat", ctypes.c_double * 3), ("ell", ctypes.c_double),
                ("e1", ctypes.c_double * 3), ("e2", ctypes.c_double * 3),
                ("a0", ctypes.c_int64), ("b0", ctypes.c_int64), ("k0", ctypes.c_int64),
                ("A", ctypes.c_int64), ("B", ctypes.c_int64), ("K", ctypes.c_int64)]


def _load_tv():
    L = _load()
    if not getattr(L, "_tv_ready", False):
        P = ctypes.POINTER
        L.orc_tv_lattice_compute.argtypes = [P(OrcGrid), P(ctypes.c_float), ctypes.c_float, P(OrcTvLattice)]
        L.orc_tv_build.argtypes = [P(OrcGrid), ctypes.c_void_p, DENSITY_FN, ctypes.c_void_p, P(OrcTvLattice),
                                   ctypes.c_float, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_tv_lookup.argtypes = [P(OrcTvLattice), ctypes.c_void_p, P(ctypes.c_float)]
        L.orc_tv_lookup.restype = ctypes.c_double
        L.orc_light_tau.argtypes = [P(OrcGrid), ctypes.c_void_p, DENSITY_FN, ctypes.c_void_p, P(ctypes.c_float),
                                    P(ctypes.c_float), ctypes.c_float, ctypes.c_double]
        L.orc_light_tau.restype = ctypes.c_double
        L._tv_ready = True
    return L


def tv_lattice(grid, Lg, hl: float) -> OrcTvLattice:
    """V2 lattice of the light step vector hl * Lg (index units)."""
    lat = OrcTvLattice()
    if _load_tv().orc_tv_lattice_compute(ctypes.byref(_grid(grid)), (ctypes.c_float * 3)(*Lg), hl, ctypes.byref(lat)):
        raise ValueError("orc_tv_lattice_compute rejected its arguments")
    return lat


def tv_build(grid, vals, lat: OrcTvLattice, hl: float, kappa: float, density_fn=None):
    """V3/V4: (tau_plus, tau_minus) as [B, K, A] float64 arrays."""
    shape = (lat.B, lat.K, lat.A)
    tp, tm = np.zeros(shape, np.float64), np.zeros(shape, np.float64)
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.float32)
    cb = DENSITY_FN(density_fn) if density_fn is not None else DENSITY_FN()
    if _load_tv().orc_tv_build(ctypes.byref(_grid(grid)), None if v is None else v.ctypes.data, cb, None,
                               ctypes.byref(lat), hl, kappa, tp.ctypes.data, tm.ctypes.data):
        raise ValueError("orc_tv_build rejected its arguments")
    return tp, tm


def tv_lookup(lat: OrcTvLattice, tau: np.ndarray, U) -> float:
    t = np.ascontiguousarray(tau, dtype=np.float64)
    return _load_tv().orc_tv_lookup(ctypes.byref(lat), t.ctypes.data, (ctypes.c_float * 3)(*U))


def light_tau(grid, vals, U, Lg, hl: float, kappa: float, density_fn=None) -> float:
    """C8's optical depth from U (the canonical light march)."""
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.float32)
    cb = DENSITY_FN(density_fn) if density_fn is not None else DENSITY_FN()
    return _load_tv().orc_light_tau(ctypes.byref(_grid(grid)), None if v is None else v.ctypes.data, cb, None,
                                    (ctypes.c_float * 3)(*U), (ctypes.c_float * 3)(*Lg), hl, kappa)

