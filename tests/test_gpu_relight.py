"""GPU parity of NEXT-2/3 relight + composite + depth shadow (R1-R3)
against oracle.relight: element by element, |gpu - oracle| <= max(1e-5 |oracle|, 1e-6)
(fp32 sums of <= 4 lights x 3 weights against fp64).  Shadow decisions are taken in
fp32 on the GPU and fp64 in the oracle; pixels whose decision margin (oracle) is below
1e-4 may differ and are only checked to be one of the two valid results."""
import math

import numpy as np
import pytest

import nsl_inputs as I
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    import paper_2604_03748_b200 as nsl
    nsl.lib()
    return nsl


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def run(nsl, cams, maps, lights, depth=None, shadow_cams=None, shadow_maps=None, **kw):
    import torch
    F, H, W = maps.shape[:3]
    out = torch.empty((F, H, W, 4), dtype=torch.float32, device="cuda")
    sm = None if shadow_maps is None else [[None if m is None else dev(m) for m in row] for row in shadow_maps]
    nsl.relight(cams, dev(maps), lights, out, depth=None if depth is None else dev(depth), shadow_cams=shadow_cams,
                shadow_maps=sm, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(F, -1, 4)


def check(g, o, margin=None, what=""):
    err = np.abs(g.astype(np.float64) - o)
    tol = np.maximum(1e-5 * np.abs(o), 1e-6)
    bad = (err > tol).any(axis=1)
    if margin is not None:
        bad &= margin >= 1e-4
    assert not bad.any(), f"{what}: {int(bad.sum())} bad, e.g. gpu {g[bad][:2]} oracle {o[bad][:2]}"


def rand_maps(seed, F, H, W):
    return np.random.default_rng(seed).random((F, H, W, 8)).astype(np.float32)


def rand_light(rng, scale=1.0):
    return I.Light(I._f32t(I._unit(tuple(rng.normal(size=3)))), I._f32t(tuple(scale * rng.random(3))))


AXIS_CAM = I.Camera(I.ORTHO, (0.5, 0.5, 2.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 1.0, 16, 12)


@pytest.mark.parametrize("to_light,chan", [((1, 0, 0), 0), ((-1, 0, 0), 4), ((0, 1, 0), 1), ((0, -1, 0), 5),
                                           ((0, 0, 1), 6), ((0, 0, -1), 2)])
def test_axis_lights_select_one_channel_exactly(nsl, to_light, chan):
    m = rand_maps(1, 1, 12, 16)
    g = run(nsl, [AXIS_CAM], m, [[I.Light(to_light, (1.0, 1.0, 1.0))]])[0]
    assert np.array_equal(g[:, 0], m.reshape(-1, 8)[:, chan])
    assert np.array_equal(g[:, 3], (1.0 - m.reshape(-1, 8)[:, 3]).astype(np.float32))


def test_worked_example_diagonal_light(nsl):
    m = np.zeros((1, 12, 16, 8), np.float32)
    m[..., 0], m[..., 1], m[..., 6] = 0.3, 0.6, 0.9
    d = 1 / math.sqrt(3)
    g = run(nsl, [AXIS_CAM], m, [[I.Light(I._f32t((d, d, d)), (1.0, 1.0, 1.0))]])[0]
    np.testing.assert_allclose(g[:, 0], (0.3 + 0.6 + 0.9) / math.sqrt(3), rtol=1e-6)


@pytest.mark.parametrize("persp", [False, True])
@pytest.mark.parametrize("n_lights", [1, 3, 4])
def test_parity_random_no_shadow(nsl, persp, n_lights):
    F, H, W = 3, 37, 53                       # ragged vs the 256-thread blocks
    rng = np.random.default_rng(10 * n_lights + persp)
    cams = [I.orbit_camera(25.0 + 40 * f, W, H, projection=I.PERSP if persp else I.ORTHO) for f in range(F)]
    lights = [[rand_light(rng) for _ in range(n_lights)] for _ in range(F)]
    m = rand_maps(n_lights, F, H, W)
    bg, emis = I._f32t((0.1, 0.2, 0.3)), I._f32t((0.7, 0.3, 0.05))
    g = run(nsl, cams, m, lights, bg=bg, emis=emis)
    for f in range(F):
        o = oracle.relight(cams[f], m[f], lights[f], bg=bg, emis=emis)["out"]
        check(g[f], o, what=f"frame {f}")


def side_scene(F=1):
    W = H = 24
    cam = I.Camera(I.ORTHO, (0.5, 2.0, 0.5), (0.0, -1.0, 0.0), (0.0, 0.0, 1.0), 1.0, W, H)
    rng = np.random.default_rng(9)
    D = (1.5 + 0.3 * rng.random((F, H, W))).astype(np.float32)
    D[rng.random((F, H, W)) < 0.2] = 0.0
    scam = I.Camera(I.ORTHO, (0.5, 0.5, 3.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 1.2, 32, 32)
    return cam, D, scam


def plate_map(scam, zp, box):
    Ws, Hs = scam.width, scam.height
    ay = scam.extent / 2
    ax = ay * Ws / Hs
    Z = np.full((Hs, Ws), np.inf, np.float32)
    for j in range(Hs):
        for i in range(Ws):
            x = scam.position[0] + (2 * (i + 0.5) / Ws - 1) * ax
            y = scam.position[1] + (1 - 2 * (j + 0.5) / Hs) * ay
            if box[0] <= x <= box[1] and box[2] <= y <= box[3]:
                Z[j, i] = scam.position[2] - zp
    return Z


def test_shadow_plate_parity(nsl):
    cam, D, scam = side_scene()
    m = rand_maps(5, 1, cam.height, cam.width)
    light = [I.Light((0.0, 0.0, 1.0), (1.0, 1.0, 1.0))]
    Z = plate_map(scam, 0.55, (0.2, 0.6, 0.3, 0.8))
    g = run(nsl, [cam], m, [light], depth=D, shadow_cams=[[scam]], shadow_maps=[[Z]])[0]
    r = oracle.relight(cam, m[0], light, depth=D[0], shadow_cams=[scam], shadow_maps=[Z])
    check(g, r["out"], r["margin"], "plate")
    lit = oracle.relight(cam, m[0], light)["out"]
    n_shadow = int((np.abs(g[:, 0]) < 0.5 * np.abs(lit[:, 0]) - 1e-6).sum())
    assert n_shadow > 10


def test_shadow_mixed_lights_persp_batch(nsl):
    """Several frames, 3 lights of which 2 carry a shadow map (one per light), a perspective
    view camera and per-frame depth with empty pixels."""
    F, W, H = 4, 40, 28
    rng = np.random.default_rng(77)
    cams = [I.orbit_camera(10.0 + 70 * f, W, H, projection=I.PERSP) for f in range(F)]
    m = rand_maps(6, F, H, W)
    D = (1.2 + 1.2 * rng.random((F, H, W))).astype(np.float32)
    D[rng.random((F, H, W)) < 0.25] = 0.0
    up = I.Light((0.0, 0.0, 1.0), (1.0, 0.9, 0.8))
    side = I.Light(I._f32t(I._unit((1.0, 0.0, 0.0))), (0.3, 0.3, 0.6))
    scam_up = I.Camera(I.ORTHO, (0.5, 0.5, 3.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 1.6, 48, 40)
    scam_side = I.Camera(I.ORTHO, (3.0, 0.5, 0.5), (-1.0, 0.0, 0.0), (0.0, 0.0, 1.0), 1.6, 32, 32)
    Zup = plate_map(scam_up, 0.6, (0.1, 0.7, 0.2, 0.9))
    Zside = np.where(rng.random((32, 32)) < 0.5, np.float32(2.0), np.float32(np.inf)).astype(np.float32)
    lights, scs, sms = [], [], []
    for f in range(F):
        lights.append([up, rand_light(rng, 0.5), side])
        scs.append([scam_up, None, scam_side])
        sms.append([Zup, None, Zside])
    g = run(nsl, cams, m, lights, depth=D, shadow_cams=scs, shadow_maps=sms, bg=(0.05, 0.05, 0.1), bias=1e-3)
    for f in range(F):
        r = oracle.relight(cams[f], m[f], lights[f], bg=(0.05, 0.05, 0.1), depth=D[f], shadow_cams=scs[f],
                           shadow_maps=sms[f], bias=1e-3)
        check(g[f], r["out"], r["margin"], f"frame {f}")


def test_parity_full_size_sampled(nsl):
    """The bench's 512x512 frames: every pixel of two frames of an 8-frame batch."""
    F, W = 8, 512
    rng = np.random.default_rng(3)
    cams = [I.orbit_camera(6.0 * f, W, W) for f in range(F)]
    lights = [[rand_light(rng) for _ in range(2)] for _ in range(F)]
    m = rand_maps(8, F, W, W)
    g = run(nsl, cams, m, lights, bg=(0.2, 0.3, 0.4))
    for f in (0, F - 1):
        check(g[f], oracle.relight(cams[f], m[f], lights[f], bg=(0.2, 0.3, 0.4))["out"], what=f"frame {f}")


def test_pipeline_bake_then_relight(nsl):
    """Six-way bake (NEXT-1) -> relight with the guiding-map depth: the GPU chain against the
    oracle fed the GPU chain's own intermediate maps (relight parity on real maps)."""
    w = I.make_workload("C1")
    b = I.default_bake(64, spp=2)
    maps = nsl.run_bake(w, b)
    rgbt, depth, _ = nsl.run_workload(w)
    import torch
    torch.cuda.synchronize()
    cam = w.cameras[0]
    light = [I.Light(I._f32t(I._unit((0.4, -0.2, 0.9))), (1.0, 0.9, 0.8))]
    out = torch.empty((1, cam.height, cam.width, 4), dtype=torch.float32, device="cuda")
    nsl.relight([cam], maps, [light], out, depth=depth, bg=(0.1, 0.1, 0.1))
    torch.cuda.synchronize()
    m8 = maps.cpu().numpy().reshape(1, cam.height, cam.width, 8)[0]
    o = oracle.relight(cam, m8, light, bg=(0.1, 0.1, 0.1))["out"]
    check(out.cpu().numpy().reshape(-1, 4), o, what="pipeline")


def test_rejects_bad_arguments(nsl):
    import torch
    m = torch.zeros((1, 4, 4, 2, 4), device="cuda")
    out = torch.empty((1, 4, 4, 4), device="cuda")
    cam = I.Camera(I.ORTHO, (0.5, 0.5, 2.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 1.0, 4, 4)
    with pytest.raises(nsl.NslError):
        nsl.relight([cam], m, [[I.Light((2.0, 0.0, 0.0), (1, 1, 1))]], out)          # not unit
    with pytest.raises(nsl.NslError):
        nsl.relight([cam], m, [[I.Light((1.0, 0.0, 0.0), (1, 1, 1))] * 5], out)      # > 4 lights
    with pytest.raises(nsl.NslError):                                              # shadow without depth
        nsl.relight([cam], m, [[I.Light((1.0, 0.0, 0.0), (1, 1, 1))]], out, shadow_cams=[[cam]],
                    shadow_maps=[[torch.zeros((4, 4), device="cuda")]])
