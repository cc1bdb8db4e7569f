"""C-ABI library checks that need no GPU: it loads, exports every entry point
include/nsl.h declares, sizes layouts, and validates arguments BEFORE any
device work (every rejection below returns NSL_ERR_INVALID_ARG with a message
and never touches CUDA)."""
import ctypes
import os
import re

import numpy as np
import pytest

import nsl_inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def nsl():
    import paper_2604_03748_b200 as nsl
    nsl.build()
    nsl.lib()
    return nsl


def header_functions():
    src = open(os.path.join(ROOT, "include", "nsl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nsl_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(nsl):
    names = header_functions()
    assert len(names) >= 10
    L = ctypes.CDLL(nsl.LIB_PATH)
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/nsl.h but not exported"
    assert set(names) == set(nsl.EXPORTS)
    assert "sm_100a" in nsl.version()


def test_library_is_sm100a_and_has_no_oracle_dependency(nsl):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", nsl.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", nsl.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "nsl_gen" not in deps


def test_product_sources_do_not_touch_the_oracle():
    pkg = os.path.join(ROOT, "paper_2604_03748_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "nsl_oracle" not in txt and "orc_" not in txt, f


def test_volume_bytes(nsl):
    g = I.Grid(4, 5, 6, (0, 0, 0), 0.25)
    lin = nsl.volume_bytes(g, nsl.LAYOUT_LINEAR_F32)
    quad = nsl.volume_bytes(g, nsl.LAYOUT_QUAD_F32)
    f16 = nsl.volume_bytes(g, nsl.LAYOUT_CORNER_F16)
    oct_ = nsl.volume_bytes(g, nsl.LAYOUT_OCT_F32)
    # body | occupancy region (2x2x2-cell blocks: 3*3*4 bits -> 4 words + 4 nbz slab words) | build scratch
    # (12 block rows x 1 flag word + 12 4-word records = 60 words) | 256-B tail: one 256-B slot each
    tail = 256 + 256 + 256
    up = lambda x: (x + 255) // 256 * 256
    assert lin == up(6 * 7 * 8 * 4) + tail
    assert quad == up(5 * 6 * 8 * 16) + tail
    assert f16 == up(5 * 6 * 7 * 16) + tail
    assert oct_ == up(5 * 6 * 7 * 32) + tail
    L = nsl.lib()
    assert L.nsl_volume_bytes(ctypes.byref(nsl.grid_desc(I.Grid(0, 5, 6, (0, 0, 0), 0.25))), 1) == 0
    assert L.nsl_volume_bytes(ctypes.byref(nsl.grid_desc(g)), 99) == 0
    # NSL_LAYOUT_AUTO (the default) resolves by size: OCT here, BRICK_OCT once the OCT body > 2 GiB
    assert nsl.layout_resolve(g, nsl.LAYOUT_AUTO) == nsl.LAYOUT_OCT_F32
    assert nsl.volume_bytes(g, nsl.LAYOUT_AUTO) == oct_
    assert nsl.layout_resolve(I.Grid(512, 512, 512, (0, 0, 0), 1 / 512), nsl.LAYOUT_AUTO) == nsl.LAYOUT_BRICK_OCT_F32
    assert nsl.layout_resolve(I.Grid(256, 256, 256, (0, 0, 0), 1 / 256), nsl.LAYOUT_AUTO) == nsl.LAYOUT_OCT_F32
    assert nsl.layout_resolve(g, nsl.LAYOUT_TEX3D_F32) == nsl.LAYOUT_TEX3D_F32
    with pytest.raises(nsl.NslError):
        nsl.volume_bytes(I.Grid(4, 5, 6, (0, 0, 0), -1.0), 1)


def _upload_rc(nsl, grid, dens, layout=1, storage=16, nbytes=1 << 20):
    h = ctypes.c_void_p()
    rc = nsl.lib().nsl_volume_upload(ctypes.byref(nsl.grid_desc(grid)), dens.ctypes.data if dens is not None else None,
                                     0, layout, storage, nbytes, None, ctypes.byref(h))
    return rc, nsl.lib().nsl_last_error().decode()


def test_upload_validation(nsl):
    g = I.Grid(4, 4, 4, (0, 0, 0), 0.25)
    ok = np.ones((4, 4, 4), np.float32)
    bad = ok.copy(); bad[1, 2, 3] = -1.0
    nan = ok.copy(); nan[0, 0, 0] = np.nan
    rc, msg = _upload_rc(nsl, g, bad)
    assert rc == 1 and "density[" in msg
    rc, msg = _upload_rc(nsl, g, nan)
    assert rc == 1 and "density[0]" in msg
    rc, msg = _upload_rc(nsl, g, ok, nbytes=16)
    assert rc == 1 and "storage_bytes" in msg
    rc, msg = _upload_rc(nsl, g, ok, storage=8)
    assert rc == 1 and "aligned" in msg
    rc, msg = _upload_rc(nsl, g, None)
    assert rc == 1
    rc, msg = _upload_rc(nsl, g, ok, layout=9)
    assert rc == 1 and "layout" in msg
    rc, msg = _upload_rc(nsl, I.Grid(4, 4, 4, (0, 0, np.inf), 0.25), ok)
    assert rc == 1 and "origin" in msg


def _batch_rc(nsl, w, **over):
    """Call nsl_guiding_map_batch with a fake (never dereferenced) volume handle: the
    call must be rejected during host validation, before any CUDA API runs."""
    cams = over.get("cams", w.cameras)
    lights = over.get("lights", w.lights)
    med = over.get("medium", w.medium)
    m = over.get("march", w.march)
    F = len(cams)
    mode = over.get("mode", w.light_mode)

    class FakeVol(ctypes.Structure):
        _fields_ = [("g", nsl.GridDesc), ("layout", ctypes.c_int32), ("data", ctypes.c_void_p), ("inv", ctypes.c_void_p)]

    fv = FakeVol(nsl.grid_desc(w.grid), 1, 4096, 4096)
    vols = (ctypes.c_void_p * 1)(ctypes.addressof(fv))
    fvol = (ctypes.c_int32 * F)(*over.get("frame_vol", [0] * F))
    cs = (nsl.CameraS * F)(*[nsl.camera_s(c) for c in cams])
    fid = (ctypes.c_uint32 * F)(*range(F))
    rc = nsl.lib().nsl_guiding_map_batch(vols, 1, fvol, cs, nsl.lights_s(lights), len(lights[0]), mode,
                                         ctypes.byref(nsl.medium_s(med)), ctypes.byref(nsl.march_s(m)), fid, F,
                                         over.get("rgbt", 4096), 4096, None, None)
    return rc, nsl.lib().nsl_last_error().decode()


def test_march_argument_validation(nsl):
    from dataclasses import replace
    w = I.make_workload("C1")
    c0 = w.cameras[0]
    cases = [
        (dict(cams=[replace(c0, forward=(0.0, 0.0, 0.5))]), "not unit"),
        (dict(cams=[replace(c0, up=c0.forward)]), "parallel"),
        (dict(cams=[replace(c0, extent=0.0)]), "extent"),
        (dict(cams=[replace(c0, width=0)]), "width"),
        (dict(cams=[replace(c0, projection=3)]), "projection"),
        (dict(medium=I.Medium(32.0, 1.5, 0.0)), "albedo"),
        (dict(medium=I.Medium(-1.0, 1.0, 0.0)), "extinction"),
        (dict(medium=I.Medium(1.0, 1.0, 1.0)), "hg_g"),
        (dict(march=replace(w.march, step=0.0)), "step"),
        (dict(march=replace(w.march, t_min=1.0)), "t_min"),
        (dict(march=replace(w.march, opacity_form=5)), "opacity_form"),
        (dict(march=replace(w.march, depth_tau=-1.0)), "depth_tau"),
        (dict(march=replace(w.march, max_steps=-2)), "max_steps"),
        (dict(march=replace(w.march, jitter=2)), "jitter"),
        (dict(march=replace(w.march, light_model=7)), "light_model"),
        (dict(lights=[[I.Light((1, 0, 0), (1, 1, 1))] * 4], mode=I.LIGHTS_GUIDE), "at most 3"),
        (dict(lights=[[I.Light((2, 0, 0), (1, 1, 1))]], mode=I.LIGHTS_EXPLICIT), "not unit"),
        (dict(lights=[[I.Light((1, 0, 0), (-1, 1, 1))]], mode=I.LIGHTS_EXPLICIT), "rgb"),
        (dict(frame_vol=[3]), "frame_vol"),
        (dict(rgbt=4100), "aligned"),
    ]
    for over, needle in cases:
        rc, msg = _batch_rc(nsl, w, **over)
        assert rc == 1, (over, msg)
        assert needle in msg, (needle, msg)


def test_relight_and_guide_lights_validation(nsl):
    """NEXT-2/3 and the guide-light helper reject bad arguments on the host, before any CUDA call."""
    L = nsl.lib()
    cam = nsl.camera_s(I.Camera(I.ORTHO, (0.5, 0.5, 2.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 1.0, 4, 4))
    f3 = ctypes.c_float * 3
    ok = nsl.lights_s([[I.Light((1.0, 0.0, 0.0), (1, 1, 1))]])
    five = nsl.lights_s([[I.Light((1.0, 0.0, 0.0), (1, 1, 1))] * 5])
    bad = nsl.lights_s([[I.Light((2.0, 0.0, 0.0), (1, 1, 1))]])
    nan_axis = f3(0, 0, float("nan"))
    cases = [
        (lambda: L.nsl_relight(ctypes.byref(cam), 1, 4096, None, five, 5, f3(0, 0, 0), f3(0, 0, 0), None, None,
                               2e-3, 4096, None), "n_lights"),
        (lambda: L.nsl_relight(ctypes.byref(cam), 1, 4096, None, bad, 1, f3(0, 0, 0), f3(0, 0, 0), None, None,
                               2e-3, 4096, None), "not unit"),
        (lambda: L.nsl_relight(ctypes.byref(cam), 1, 4100, None, ok, 1, f3(0, 0, 0), f3(0, 0, 0), None, None,
                               2e-3, 4096, None), "aligned"),
        (lambda: L.nsl_relight(ctypes.byref(cam), 1, 4096, None, ok, 1, f3(0, 0, 0), f3(0, 0, 0), None, None,
                               -1.0, 4096, None), "bias"),
        (lambda: L.nsl_relight(ctypes.byref(cam), 0, 4096, None, ok, 1, f3(0, 0, 0), f3(0, 0, 0), None, None,
                               2e-3, 4096, None), "F"),
        (lambda: L.nsl_guide_lights(None, None, None, None, None), "NULL"),
        (lambda: L.nsl_guide_lights(ctypes.byref(cam), ctypes.addressof(nan_axis), None, (nsl.LightS * 3)(), None),
         "axis"),
    ]
    for call, needle in cases:
        rc = call()
        msg = L.nsl_last_error().decode()
        assert rc == 1, (needle, msg)
        assert needle in msg, (needle, msg)


def test_animated_validation(nsl):
    """nsl_guiding_map_animated checks every frame's storage, camera and light before enqueuing."""
    from dataclasses import replace
    L = nsl.lib()
    w = I.make_workload("C1")
    g = nsl.grid_desc(w.grid)
    nb = nsl.volume_bytes(w.grid, 3)
    F = 2
    cams = (nsl.CameraS * F)(*[nsl.camera_s(w.cameras[0])] * F)
    bad_cams = (nsl.CameraS * F)(nsl.camera_s(w.cameras[0]), nsl.camera_s(replace(w.cameras[0], width=0)))
    ls = nsl.lights_s([w.lights[0]] * F)
    med, mar = nsl.medium_s(w.medium), nsl.march_s(w.march)
    fid = (ctypes.c_uint32 * F)(0, 1)
    vp2 = ctypes.c_void_p * F

    def call(dens=(4096, 4096), stor=(8192, 8192), nbytes=nb, cs=cams, f=F, chunk=0, rgbt=4096):
        return L.nsl_guiding_map_animated(ctypes.byref(g), vp2(*dens), 3, vp2(*stor), nbytes, cs, ls,
                                          len(w.lights[0]), w.light_mode, ctypes.byref(med), ctypes.byref(mar),
                                          fid, f, chunk, rgbt, 4096, None, None)
    cases = [
        (dict(dens=(4096, 0)), "NULL density of frame 1"),
        (dict(stor=(8192, 0)), "NULL storage"),
        (dict(stor=(8192, 8200)), "aligned"),
        (dict(nbytes=nb - 1), "storage_bytes"),
        (dict(cs=bad_cams), "width"),
        (dict(f=0), "F must be"),
        (dict(chunk=-1), "chunk"),
        (dict(rgbt=4100), "aligned"),
    ]
    for over, needle in cases:
        rc = call(**over)
        msg = L.nsl_last_error().decode()
        assert rc == 1, (over, msg)
        assert needle in msg, (needle, msg)


def test_bench_l1_gather_validation(nsl):
    L = nsl.lib()
    n = ctypes.c_uint64()
    for args, needle in [((None, 1, 1, 4096, 1 << 20), "NULL"), ((4096, 0, 1, 4096, 1 << 20), "waves")]:
        vol, waves, reps, sink, nf = args
        rc = L.nsl_bench_l1_gather(vol, waves, reps, sink, nf, ctypes.byref(n), None)
        msg = L.nsl_last_error().decode()
        assert rc == 1 and needle in msg, (args, msg)


def test_mixed_sizes_rejected(nsl):
    from dataclasses import replace
    w = I.make_workload("C2", frames=[0, 1])
    cams = [w.cameras[0], replace(w.cameras[1], width=256)]
    rc, msg = _batch_rc(nsl, w, cams=cams)
    assert rc == 1 and "size differs" in msg


def test_binding_has_no_fallback(monkeypatch, nsl):
    monkeypatch.setattr(nsl, "_lib", None)
    monkeypatch.setattr(nsl, "LIB_PATH", "/nonexistent/libnsl.so")
    with pytest.raises(nsl.NslError):
        nsl.lib()


def test_c_example_compiles_as_c99(tmp_path):
    """The boundary is plain C: examples/guiding_map_c.c builds with gcc -std=c99 -Wall -Werror
    against include/nsl.h and links against libnsl.so (no CUDA headers, no Python)."""
    import subprocess
    import paper_2604_03748_b200 as nsl
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = nsl.build()                      # the library in use (NSL_LIB may point at a build variant)
    libdir = os.path.dirname(lib)
    exe = tmp_path / "gm"
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", "guiding_map_c.c"), lib,
                           f"-Wl,-rpath,{libdir}", "-lm", "-o", str(exe)])
    assert exe.exists()
