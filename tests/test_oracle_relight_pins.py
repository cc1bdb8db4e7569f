"""Pins of the relight / composite / depth-shadow oracle (NEXT-2/3):
axis exactness, the worked example (0.3+0.6+0.9)/sqrt(3), linearity and
additivity over lights, transparency-only composite, and the shadow test against a
brute-force geometric occluder check."""
import math

import numpy as np
import pytest

import nsl_inputs as I

AXIS_CAM = I.Camera(I.ORTHO, (0.5, 0.5, 2.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 1.0, 16, 12)


def maps(seed=0, H=12, W=16):
    return np.random.default_rng(seed).random((H, W, 8)).astype(np.float32)


@pytest.mark.parametrize("to_light,chan", [((1, 0, 0), 0), ((-1, 0, 0), 4), ((0, 1, 0), 1), ((0, -1, 0), 5),
                                           ((0, 0, 1), 6), ((0, 0, -1), 2)])
def test_axis_lights_select_one_channel_exactly(orc, to_light, chan):
    m = maps(1)
    r = orc.relight(AXIS_CAM, m, [I.Light(to_light, (1.0, 1.0, 1.0))])
    # to_light +x = right (L_x+), +y = top, +z = toward the camera = front; -z = back
    assert np.array_equal(r["out"][:, 0], m.reshape(-1, 8)[:, chan].astype(np.float64))
    assert np.array_equal(r["out"][:, 3], 1.0 - m.reshape(-1, 8)[:, 3].astype(np.float64))


def test_worked_example_diagonal_light(orc):
    m = np.zeros((12, 16, 8), np.float32)
    m[..., 0], m[..., 1], m[..., 6] = 0.3, 0.6, 0.9          # right, top, front
    d = 1 / math.sqrt(3)
    r = orc.relight(AXIS_CAM, m, [I.Light((d, d, d), (1.0, 1.0, 1.0))])
    np.testing.assert_allclose(r["out"][:, 0], (0.3 + 0.6 + 0.9) / math.sqrt(3), rtol=1e-6)   # 1.0392
    w = orc.relight_weights(AXIS_CAM, [I.Light((d, d, d), (1, 1, 1))])
    assert 1.0 <= np.abs(w).sum() <= math.sqrt(3) + 1e-6


def test_weights_l1_norm_between_1_and_sqrt3(orc):
    rng = np.random.default_rng(3)
    cam = I.orbit_camera(37.0, 8, 8)
    for _ in range(200):
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        w = orc.relight_weights(cam, [I.Light(tuple(v), (1, 1, 1))])
        s = np.abs(w).sum()
        assert 1.0 - 1e-6 <= s <= math.sqrt(3) + 1e-6


def test_linearity_additivity_and_transparency_only(orc):
    m = maps(2)
    cam = I.orbit_camera(20.0, 16, 12)
    L = I._f32t(I._unit((0.3, -0.4, 0.7)))
    one = orc.relight(cam, m, [I.Light(L, (1.0, 0.5, 0.25))])["out"]
    two = orc.relight(cam, m, [I.Light(L, (0.5, 0.25, 0.125)), I.Light(L, (0.5, 0.25, 0.125))])["out"]
    np.testing.assert_allclose(two, one, rtol=1e-12)
    bg = (0.2, 0.4, 0.8)
    dark = orc.relight(cam, m, [I.Light(L, (0.0, 0.0, 0.0))], bg=bg)["out"]
    np.testing.assert_allclose(dark[:, :3], m.reshape(-1, 8)[:, 3:4] * np.array(bg, np.float32), rtol=1e-7)
    em = orc.relight(cam, m, [I.Light(L, (0.0, 0.0, 0.0))], emis=(1.0, 0.5, 0.0))["out"]
    np.testing.assert_allclose(em[:, 1], 0.5 * m.reshape(-1, 8)[:, 7], rtol=1e-7)


def side_scene():
    """Camera looking along -y at the unit box; light from +z with an orthographic shadow
    camera above; synthetic smoke-shell depths D (some pixels empty)."""
    W = H = 24
    cam = I.Camera(I.ORTHO, (0.5, 2.0, 0.5), (0.0, -1.0, 0.0), (0.0, 0.0, 1.0), 1.0, W, H)
    rng = np.random.default_rng(9)
    D = (1.5 + 0.3 * rng.random((H, W))).astype(np.float32)
    D[rng.random((H, W)) < 0.2] = 0.0
    scam = I.Camera(I.ORTHO, (0.5, 0.5, 3.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 1.2, 32, 32)
    return cam, D, scam


def plate_map(scam, zp, box):
    """Depth map of a horizontal plate at height zp over [x0,x1]x[y0,y1] seen from scam."""
    Ws, Hs = scam.width, scam.height
    ay = scam.extent / 2
    ax = ay * Ws / Hs
    Z = np.full((Hs, Ws), np.inf, np.float32)
    for j in range(Hs):
        for i in range(Ws):
            x = scam.position[0] + (2 * (i + 0.5) / Ws - 1) * ax      # shadow camera: r = +x, u = +y
            y = scam.position[1] + (1 - 2 * (j + 0.5) / Hs) * ay
            if box[0] <= x <= box[1] and box[2] <= y <= box[3]:
                Z[j, i] = scam.position[2] - zp
    return Z


def test_shadow_plate_matches_geometric_brute_force(orc):
    cam, D, scam = side_scene()
    m = np.ones((cam.height, cam.width, 8), np.float32)
    m[..., 3] = 0.0
    light = [I.Light((0.0, 0.0, 1.0), (1.0, 1.0, 1.0))]
    zp, box, bias = 0.55, (0.2, 0.6, 0.3, 0.8), 2e-3
    Z = plate_map(scam, zp, box)
    r = orc.relight(cam, m, light, depth=D, shadow_cams=[scam], shadow_maps=[Z], bias=bias)
    lit = orc.relight(cam, m, light, depth=D)["out"][:, 0]
    vis = r["out"][:, 0] / lit
    # brute force: shell point p = origin + D * (0,-1,0); shadowed iff the map cell above p is
    # covered by the plate and p lies below the plate by more than the bias
    Ws, Hs = scam.width, scam.height
    ay = scam.extent / 2
    ax = ay * Ws / Hs
    n_shadow = 0
    for py in range(cam.height):
        for px in range(cam.width):
            q = py * cam.width + px
            if D[py, px] == 0 or r["margin"][q] < 1e-6:
                continue
            x = 0.5 - (2 * (px + 0.5) / cam.width - 1) * 0.5     # screen right = f x up = -x
            z = 0.5 + (1 - 2 * (py + 0.5) / cam.height) * 0.5
            i = math.floor(((x - 0.5) / ax + 1) * Ws / 2)
            j = math.floor((1 - (2.0 - D[py, px] - 0.5) / ay) * Hs / 2)
            covered = 0 <= i < Ws and 0 <= j < Hs and np.isfinite(Z[j, i])
            expect = 0.0 if (covered and z < zp - bias) else 1.0
            assert vis[q] == expect, (px, py, vis[q], expect)
            n_shadow += expect == 0.0
    assert n_shadow > 10


def test_shadow_empty_map_and_plate_behind(orc):
    cam, D, scam = side_scene()
    m = maps(4, cam.height, cam.width)
    light = [I.Light((0.0, 0.0, 1.0), (1.0, 1.0, 1.0))]
    free = orc.relight(cam, m, light, depth=D)["out"]
    empty = orc.relight(cam, m, light, depth=D, shadow_cams=[scam],
                        shadow_maps=[np.full((32, 32), np.inf, np.float32)])["out"]
    assert np.array_equal(free, empty)
    behind = orc.relight(cam, m, light, depth=D, shadow_cams=[scam],
                         shadow_maps=[plate_map(scam, -0.5, (0, 1, 0, 1))])["out"]   # plate below all smoke
    assert np.array_equal(free, behind)
