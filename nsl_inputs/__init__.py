"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the guiding-map method's arithmetic (DESIGN.md
§"Oracle independence"): it manufactures density grids (via the small C
generator ``gen.c``), camera paths, explicit light lists and parameter
records shaped like the paper's scenes, exactly as DESIGN.md §"Input recipe"
states.  Guide-light frames, frame constants, jitter, sampling and every
other step of Algorithm 1 are implemented separately and
independently by ``oracle/`` and by ``paper_2604_03748_b200``.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB_PATH = os.path.join(_HERE, "libnsl_gen.so")
_lib = None

KINDS = {"puff": 0, "plume": 1, "carved": 2, "const": 3}


def build(force: bool = False) -> str:
    """Compile gen.c into libnsl_gen.so (in-tree)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.nslgen_volume.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_uint32, ctypes.c_int,
                                      ctypes.c_void_p]
        lib.nslgen_volume.restype = ctypes.c_int
        lib.nslgen_fnv1a64.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        lib.nslgen_fnv1a64.restype = ctypes.c_uint64
        _lib = lib
    return _lib


def volume(kind: str, n: int, frame: float = 0.0, seed: int = 0x26040374,
           dims: Optional[Sequence[int]] = None, threads: Optional[int] = None) -> np.ndarray:
    """Density grid, float32 array shaped [nz, ny, nx] (x fastest), values in [0,1]."""
    nx, ny, nz = dims if dims is not None else (n, n, n)
    out = np.empty((nz, ny, nx), dtype=np.float32)
    if threads is None:
        threads = min(os.cpu_count() or 1, 64)
    rc = _load().nslgen_volume(KINDS[kind], nx, ny, nz, float(frame), seed & 0xFFFFFFFF, threads,
                               out.ctypes.data)
    if rc != 0:
        raise ValueError(f"nslgen_volume failed for kind={kind}")
    return out


def content_hash(arr: np.ndarray) -> str:
    a = np.ascontiguousarray(arr)
    return "%016x" % _load().nslgen_fnv1a64(a.ctypes.data, a.nbytes)


# --------------------------------------------------------------------------
# Parameter records (plain data; each side marshals them into its own structs)
# --------------------------------------------------------------------------
ORTHO, PERSP = 0, 1
LIGHTS_EXPLICIT, LIGHTS_GUIDE = 0, 1
EXP, RIEMANN, LITERAL = 0, 1, 2


@dataclass
class Grid:
    nx: int
    ny: int
    nz: int
    origin: tuple = (0.0, 0.0, 0.0)
    voxel_width: float = 1.0


@dataclass
class Camera:
    projection: int
    position: tuple
    forward: tuple
    up: tuple
    extent: float          # ortho: image-plane height (world); persp: 2*tan(fov_y/2)
    width: int
    height: int


@dataclass
class Light:
    to_light: tuple        # unit, scene -> light (ignored in guide mode)
    rgb: tuple


@dataclass
class Medium:
    extinction: float      # kappa: sigma_t = kappa * rho
    albedo: float          # alpha: sigma_s = alpha * sigma_t
    hg_g: float = 0.0


@dataclass
class March:
    step: float            # h (world units)
    light_step: float = 0.0   # h_l; 0 -> h
    max_steps: int = 0        # N; 0 -> until the support exit
    depth_tau: float = -1.0   # tau vs sigma_s; <0 -> default 0.01*alpha*kappa (set by scene)
    t_min: float = 1e-4
    opacity_form: int = EXP
    jitter: int = 1
    seed: int = 0x26040374
    guide_axis: tuple = (0.0, 0.0, 1.0)
    front_identity: int = 1   # allow the GPU front-light shortcut (C9); oracle ignores
    light_model: int = 0      # 0 canonical light march (C8), 1 transmittance volume


@dataclass
class Bake:
    """Six-way bake parameters: spp, primary step h_b, light step h_bl (world)."""
    spp: int = 16
    step: float = 0.0
    light_step: float = 0.0
    max_steps: int = 0
    t_min: float = 1e-4
    seed: int = 0x6B616B65


def default_bake(n: int, spp: int = 16, **kw) -> "Bake":
    b = Bake(spp=spp, step=float(np.float32(1.0 / n)), light_step=float(np.float32(2.0 / n)))
    return replace(b, **kw)


@dataclass
class Workload:
    name: str
    grid: Grid
    volume_specs: List[tuple]          # per distinct volume: (kind, frame_t)
    frame_vol: List[int]               # F -> index into volume_specs
    cameras: List[Camera]
    light_mode: int
    lights: List[List[Light]]          # F x n_lights
    medium: Medium
    march: March
    frame_ids: List[int]
    seed: int = 0x26040374
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def n_frames(self) -> int:
        return len(self.cameras)

    @property
    def n_lights(self) -> int:
        return len(self.lights[0])

    @property
    def width(self) -> int:
        return self.cameras[0].width

    @property
    def height(self) -> int:
        return self.cameras[0].height

    def volume(self, idx: int) -> np.ndarray:
        if idx not in self._cache:
            kind, t = self.volume_specs[idx]
            g = self.grid
            self._cache[idx] = volume(kind, g.nx, frame=t, seed=self.seed, dims=(g.nx, g.ny, g.nz))
        return self._cache[idx]

    def subset(self, frames: Sequence[int]) -> "Workload":
        """The same workload restricted to the listed global frames (volumes re-indexed)."""
        frames = list(frames)
        vols = sorted(set(self.frame_vol[f] for f in frames))
        remap = {v: i for i, v in enumerate(vols)}
        w = replace(self,
                    volume_specs=[self.volume_specs[v] for v in vols],
                    frame_vol=[remap[self.frame_vol[f]] for f in frames],
                    cameras=[self.cameras[f] for f in frames],
                    lights=[self.lights[f] for f in frames],
                    frame_ids=[self.frame_ids[f] for f in frames],
                    _cache={})
        for v in vols:
            if v in self._cache:
                w._cache[remap[v]] = self._cache[v]
        return w


def _unit(v):
    n = math.sqrt(sum(c * c for c in v))
    return tuple(c / n for c in v)


def orbit_camera(yaw_deg: float, width: int, height: int, elev_deg: float = 15.0,
                 distance: float = 2.0, extent: float = 1.8, projection: int = ORTHO,
                 fov_deg: float = 40.0, target=(0.5, 0.5, 0.5)) -> Camera:
    """Camera orbiting the unit box about the world z axis (z up)."""
    yaw, el = math.radians(yaw_deg), math.radians(elev_deg)
    d = (math.cos(el) * math.cos(yaw), math.cos(el) * math.sin(yaw), math.sin(el))
    pos = tuple(t + distance * c for t, c in zip(target, d))
    fwd = _unit(tuple(-c for c in d))
    if projection == PERSP:
        extent = 2.0 * math.tan(math.radians(fov_deg) / 2.0)
    f32 = lambda v: tuple(float(np.float32(c)) for c in v)
    return Camera(projection, f32(pos), f32(fwd), (0.0, 0.0, 1.0), float(np.float32(extent)),
                  width, height)


def default_march(n: int, cfg_index: int, medium: Medium, **kw) -> March:
    h = float(np.float32(10.0 / n))            # h = 10 dx
    m = March(step=h, light_step=0.0, depth_tau=float(np.float32(0.01 * medium.albedo * medium.extinction)),
              seed=0x26040374 + cfg_index)
    return replace(m, **kw)


def _f32t(v):
    return tuple(float(np.float32(c)) for c in v)


WHITE = (1.0, 1.0, 1.0)


def guide_lights(rgb=(WHITE, WHITE, WHITE)) -> List[Light]:
    return [Light((0.0, 0.0, 0.0), tuple(c)) for c in rgb]


def make_workload(cfg: str, frames: Optional[Sequence[int]] = None, kappa: float = 32.0,
                  perspective: bool = False, single_light: bool = False,
                  light_set: str = "guide") -> Workload:
    """The configs of BASELINE.json (C1..C5) per DESIGN.md §"Input recipe", and P482: the
    paper's own timed workload (§5 Performance: a 512^2 guiding map over a 400^3
    density grid, h = 10 dx, the three surrogate lights; one frame per simulation step), on the
    C2 plume recipe and camera path."""
    medium = Medium(extinction=kappa, albedo=1.0, hg_g=0.0)
    idx = {"C1": 0, "C2": 1, "C3": 2, "C4": 3, "C5": 4, "P482": 5}[cfg]
    seed = 0x26040374 + idx
    if cfg == "C1":
        n, res, F = 64, 128, 1
        cams = [orbit_camera(30.0, res, res, projection=PERSP if perspective else ORTHO)]
        specs, fvol = [("puff", 0.0)], [0]
        if single_light:
            mode = LIGHTS_EXPLICIT
            lights = [[Light(_f32t(_unit((0.3, -0.5, 0.8))), (1.0, 0.95, 0.9))]]
        else:
            mode = LIGHTS_GUIDE
            lights = [guide_lights() if light_set == "guide" else guide_lights((WHITE,))]
    elif cfg == "C2":
        n, res, F = 128, 512, 60
        cams = [orbit_camera(6.0 * f, res, res) for f in range(F)]
        specs, fvol = [("plume", 0.0)], [0] * F
        mode, lights = LIGHTS_GUIDE, [guide_lights() for _ in range(F)]
    elif cfg == "C3":
        n, res, F = 256, 1024, 60
        cams = [orbit_camera(30.0, res, res) for _ in range(F)]
        specs, fvol = [("carved", 0.0)], [0] * F
        mode = LIGHTS_EXPLICIT
        lights = []
        for f in range(F):
            a, e = math.radians(6.0 * f), math.radians(35.0)
            lights.append([Light(_f32t(_unit((math.cos(a) * math.cos(e), math.sin(a) * math.cos(e),
                                               math.sin(e)))), (1.0, 0.85, 0.7))])
    elif cfg == "C4":
        n, res, F = 256, 1024, 240
        cams = [orbit_camera(1.5 * f, res, res) for f in range(F)]
        specs, fvol = [("plume", float(f)) for f in range(F)], list(range(F))
        mode, lights = LIGHTS_GUIDE, [guide_lights() for _ in range(F)]
    elif cfg == "P482":
        n, res, F = 400, 512, 60
        cams = [orbit_camera(6.0 * f, res, res) for f in range(F)]
        specs, fvol = [("plume", 0.0)], [0] * F
        mode, lights = LIGHTS_GUIDE, [guide_lights() for _ in range(F)]
    elif cfg == "C5":
        n, res, F = 512, 2048, 1024
        cams = [orbit_camera(360.0 * f / 1024.0, res, res) for f in range(F)]
        specs, fvol = [("plume", 0.0)], [0] * F
        mode, lights = LIGHTS_GUIDE, [guide_lights() for _ in range(F)]
    else:
        raise ValueError(cfg)
    grid = Grid(n, n, n, (0.0, 0.0, 0.0), float(np.float32(1.0 / n)))
    w = Workload(name=cfg, grid=grid, volume_specs=specs, frame_vol=fvol, cameras=cams,
                 light_mode=mode, lights=lights, medium=medium,
                 march=default_march(n, idx, medium), frame_ids=list(range(F)), seed=seed)
    if frames is not None:
        w = w.subset(frames)
    return w
