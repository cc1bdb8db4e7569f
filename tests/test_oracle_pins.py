"""Pins of the CPU oracle against values fixed by the paper and by mathematics.

Every test here checks oracle/ against something other than itself
(DESIGN.md §4 "Pins"): closed forms of Algorithm 1 on analytic media
(slab P2, sphere P3, constant grid P4), invariants (conservation P5, bounds
P6, linearity P7, mirror symmetry P8), brute force (P9 opaque voxel, P10
clip-free loop, P11 continuum convergence, P13 sampler), textbook values
(P12 Henyey-Greenstein, P14 MurmurHash3 fmix32).  All CPU, marker "not gpu".
"""
import math

import numpy as np
import pytest

import nsl_inputs as I

FOUR_PI = 4.0 * math.pi


# --------------------------------------------------------------------------- helpers
def grid64(n=64, nz=None):
    return I.Grid(n, n, nz or n, (0.0, 0.0, 0.0), float(np.float32(1.0 / n)))


def cam_down(W=32, H=32, z=2.0, extent=0.9, x=0.5, y=0.5, proj=I.ORTHO):
    """Orthographic camera above the box looking along -z; screen right = +x, up = +y."""
    return I.Camera(proj, (x, y, z), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), extent, W, H)


def march(h, **kw):
    base = dict(step=h, light_step=0.0, max_steps=0, depth_tau=0.0, t_min=0.0, opacity_form=I.EXP,
                jitter=0, seed=1234, guide_axis=(0.0, 0.0, 1.0))
    base.update(kw)
    return I.March(**base)


FRONT_DOWN = [I.Light((0.0, 0.0, 1.0), (1.0, 1.0, 1.0))]    # to_light = -forward


def pixel_index_coords(cam, grid, px, py):
    """Independent fp64 evaluation of the orthographic pixel-ray origin in
    padded index space: u = (p - o)/dx + 1/2, p = P + s_x a_x r + s_y a_y u."""
    W, H = cam.width, cam.height
    sx = 2.0 * (px + 0.5) / W - 1.0
    sy = 1.0 - 2.0 * (py + 0.5) / H
    ay = cam.extent / 2.0
    ax = ay * W / H
    # r = +x, u = +y for cam_down
    wx = cam.position[0] + sx * ax
    wy = cam.position[1] + sy * ay
    return wx / grid.voxel_width + 0.5, wy / grid.voxel_width + 0.5


def slab_closed_form(s, k, form, alpha, P, h):
    """Discrete Alg.-1 sums for k equal samples of optical thickness s, front light retracing the view ray."""
    e2 = math.exp(-2.0 * s * k)
    if form == I.EXP:
        return P * alpha * (1.0 - e2) / (1.0 + math.exp(-s))
    riemann = P * alpha * s * (1.0 - e2) / (1.0 - math.exp(-2.0 * s))
    if form == I.RIEMANN:
        return riemann
    return riemann / h                 # LITERAL: A_n = T_{n-1} sigma_s (no h)


# --------------------------------------------------------------------------- P12, P14, P13
def test_hg_textbook_values(orc):
    assert orc.hg(0.0, 0.3) == pytest.approx(1.0 / FOUR_PI, rel=1e-15)           # isotropic
    assert orc.hg(0.5, 1.0) == pytest.approx(0.75 / (FOUR_PI * 0.125), rel=1e-15)
    assert orc.hg(0.5, 1.0) == pytest.approx(0.477465, abs=1e-6)
    from scipy.integrate import quad
    for g in (-0.8, -0.3, 0.0, 0.3, 0.8):
        total = 2.0 * math.pi * quad(lambda c: orc.hg(g, c), -1.0, 1.0, epsabs=1e-12)[0]
        assert total == pytest.approx(1.0, abs=1e-6)                                 # normalised
        mean_cos = 2.0 * math.pi * quad(lambda c: c * orc.hg(g, c), -1.0, 1.0, epsabs=1e-12)[0]
        assert mean_cos == pytest.approx(g, abs=1e-6)                                # <cos> = g


def test_fmix32_published_values(orc):
    # MurmurHash3 fmix32: fmix32(0) = 0 and fmix32(1) = 0x514E28B7 (published finaliser output)
    assert orc.fmix32(0) == 0
    assert orc.fmix32(1) == 0x514E28B7


def test_jitter_range_and_uniformity(orc):
    m = march(0.15625, jitter=1, seed=0x26040374)
    d = np.array([orc.jitter_delta(m, 7, p) for p in range(20000)])
    assert d.min() >= 0.0 and d.max() < m.step
    # uniform on [0, h): mean h/2, variance h^2/12 (4-sigma bands)
    assert abs(d.mean() - m.step / 2) < 4 * m.step / math.sqrt(12 * 20000)
    assert d.var() == pytest.approx(m.step ** 2 / 12, rel=0.05)
    assert orc.jitter_delta(march(0.15625, jitter=0), 7, 5) == 0.0
    # keyed by (seed, frame, pixel): changing any key changes the value
    assert orc.jitter_hash(1, 2, 3) != orc.jitter_hash(1, 2, 4)
    assert orc.jitter_hash(1, 2, 3) != orc.jitter_hash(1, 3, 3)
    assert orc.jitter_hash(1, 2, 3) != orc.jitter_hash(1 | (1 << 40), 2, 3)


def test_sampler_voxel_centres_constants_midpoint(orc):
    rng = np.random.default_rng(0)
    g = I.Grid(5, 4, 3, (0, 0, 0), 0.25)
    v = rng.random((3, 4, 5)).astype(np.float32)
    for (i, j, k) in [(0, 0, 0), (4, 3, 2), (2, 1, 1)]:
        # voxel (i,j,k) sits at padded index u = (i+1, j+1, k+1): exact value
        assert orc.sample(g, v, (i + 1.0, j + 1.0, k + 1.0)) == float(v[k, j, i])
    c = np.full((3, 4, 5), 0.5, np.float32)
    for u in [(1.0, 1.0, 1.0), (2.3, 2.9, 2.5), (4.99, 3.5, 1.01)]:
        assert orc.sample(g, c, u) == pytest.approx(0.5, abs=1e-15)      # constant interior
    g2 = I.Grid(2, 1, 1, (0, 0, 0), 1.0)
    v2 = np.array([[[0.0, 1.0]]], np.float32)
    assert orc.sample(g2, v2, (1.5, 1.0, 1.0)) == pytest.approx(0.5, abs=1e-15)  # midpoint
    # border-zero apron: half-way into the apron is half the boundary value; outside support = 0
    assert orc.sample(g2, v2, (0.5, 1.0, 1.0)) == pytest.approx(0.0)
    assert orc.sample(g2, v2, (2.5, 1.0, 1.0)) == pytest.approx(0.5)
    assert orc.sample(g2, v2, (3.0, 1.0, 1.0)) == 0.0
    assert orc.sample(g2, v2, (0.0, 1.0, 1.0)) == 0.0


def _trilinear_np(vals, u):
    """Independent fp64 trilinear with a zero apron (weights form, not lerp form)."""
    nz, ny, nx = vals.shape
    pad = np.zeros((nz + 2, ny + 2, nx + 2))
    pad[1:-1, 1:-1, 1:-1] = vals
    u = np.asarray(u, np.float64)
    out = np.zeros(len(u))
    ok = np.all((u > 0) & (u < np.array([nx + 1, ny + 1, nz + 1])), axis=1)
    i0 = np.floor(u[ok]).astype(int)
    f = u[ok] - i0
    acc = np.zeros(ok.sum())
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                w = (f[:, 0] if dx else 1 - f[:, 0]) * (f[:, 1] if dy else 1 - f[:, 1]) * (f[:, 2] if dz else 1 - f[:, 2])
                acc += w * pad[i0[:, 2] + dz, i0[:, 1] + dy, i0[:, 0] + dx]
    out[ok] = acc
    return out


def test_sampler_matches_weights_form_brute_force(orc):
    rng = np.random.default_rng(1)
    g = I.Grid(6, 5, 7, (0, 0, 0), 0.1)
    v = rng.random((7, 5, 6)).astype(np.float32)
    u = (rng.random((500, 3)) * np.array([8.0, 7.0, 9.0]) - 0.5).astype(np.float32)
    ref = _trilinear_np(v, u.astype(np.float64))
    got = np.array([orc.sample(g, v, tuple(x)) for x in u])
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-14)


# --------------------------------------------------------------------------- P1 zero grid
def test_zero_grid(orc):
    w = I.make_workload("C1")
    vals = np.zeros_like(w.volume(0))
    r = orc.guiding_map(w.grid, vals, w.cameras[0], w.lights[0], w.light_mode, w.medium, w.march)
    assert np.all(r["rgbt"][:, :3] == 0.0) and np.all(r["rgbt"][:, 3] == 1.0)
    assert np.all(r["depth"] == 0.0)
    d = r["debug"]
    assert np.all(d[:, 2] == 0) and np.all(d[:, 4] == 0) and np.all(d[:, 5] == 0)
    assert np.any(d[:, 0] > 0)                       # rays do cross the support
    assert np.all(d[:, 3] == d[:, 1])                # no early termination: n_term = n_hi


# --------------------------------------------------------------------------- P2 homogeneous slab
@pytest.mark.parametrize("form", [I.EXP, I.RIEMANN, I.LITERAL])
@pytest.mark.parametrize("zlo,zhi,rho0,kappa,alpha,g", [
    (20.0, 50.0, 0.7, 3.0, 1.0, 0.0),
    (5.0, 61.0, 1.3, 0.9, 0.6, 0.3),
    (30.0, 40.0, 2.0, 10.0, 0.8, -0.5),
])
def test_slab_closed_form(orc, form, zlo, zhi, rho0, kappa, alpha, g):
    kappa, alpha, g = (float(np.float32(x)) for x in (kappa, alpha, g))   # the ABI carries fp32
    grid = grid64()
    cam = cam_down(W=16, H=16, extent=0.9)
    h = 0.15625                           # 10 dx at dx = 1/64; samples at U_z = 128.5 - 10 n
    slab = lambda u, ctx: rho0 if zlo < u[2] < zhi else 0.0
    med = I.Medium(kappa, alpha, g)
    r = orc.guiding_map(grid, None, cam, FRONT_DOWN, I.LIGHTS_EXPLICIT, med, march(h, opacity_form=form),
                        density_fn=slab)
    zs = 128.5 - 10.0 * np.arange(1, 14)
    k = int(np.sum((zs > zlo) & (zs < zhi)))
    s = kappa * rho0 * h                  # optical thickness of one step (sigma_t = kappa rho)
    P = (1 - g * g) / (FOUR_PI * (1 + g) ** 3)   # HG at cos = -1 (front light backscatter)
    np.testing.assert_allclose(r["rgbt"][:, 3], math.exp(-s * k), rtol=1e-13)
    np.testing.assert_allclose(r["rgbt"][:, 0], slab_closed_form(s, k, form, alpha, P, h), rtol=1e-12)
    # depth: first sample inside the slab (sigma_s = alpha kappa rho0 > tau = 0), D = t_n = n h
    n_first = int(np.argmax((zs > zlo) & (zs < zhi))) + 1
    assert np.all(r["depth"] == np.float32(n_first * h))


def test_slab_side_lights_closed_form(orc):
    """Guide set on a z-slab seen from above: the side lights (omega x z) are horizontal here
    because the guide axis is chosen as +y; each side march stays inside the slab and its
    transmittance is exp(-kappa rho0 h_l M) with M the in-support sample count."""
    grid = grid64()
    W = H = 8
    cam = cam_down(W=W, H=H, extent=0.5)
    h = 0.15625
    rho0, kappa = 0.5, 2.0
    slab = lambda u, ctx: rho0 if 20.0 < u[2] < 50.0 else 0.0
    m = march(h, guide_axis=(0.0, 1.0, 0.0))
    lights = I.guide_lights()
    r = orc.guiding_map(grid, None, cam, lights, I.LIGHTS_GUIDE, I.Medium(kappa, 1.0, 0.0), m, density_fn=slab)
    fc = orc.frame_constants(grid, cam, lights, I.LIGHTS_GUIDE, I.Medium(kappa, 1.0, 0.0), m)
    # omega = +z, axis = +y: omega x y = (0*0 - 1*1, ..) = (-1, 0, 0)
    np.testing.assert_allclose(fc["Ln"], [[0, 0, 1], [-1, 0, 0], [1, 0, 0]], atol=1e-7)
    s = kappa * rho0 * h
    P = 1.0 / FOUR_PI
    for q in range(W * H):
        px, py = q % W, q // W
        ux, _ = pixel_index_coords(cam, grid, px, py)
        # side samples at ux -/+ 10 j; in support while 0 < x < 65
        M_left = int(np.floor((ux - 1e-9) / 10.0))          # ux - 10 j > 0
        M_right = int(np.floor((65.0 - ux - 1e-9) / 10.0))  # ux + 10 j < 65
        Tl, Tr = math.exp(-s * M_left), math.exp(-s * M_right)
        k = 3
        A = [math.exp(-s * i) * (1 - math.exp(-s)) for i in range(k)]
        front = sum(a * math.exp(-s * i) for i, a in enumerate(A))
        expect = P * (front + sum(A) * (Tl + Tr))
        assert r["rgbt"][q, 0] == pytest.approx(expect, rel=1e-12)
        # front marches from z = 48.5/38.5/28.5 up to z < 65 take 1, 2, 3 samples
        assert r["debug"][q, 5] == 6 + k * (M_left + M_right)
    d = r["debug"]
    assert np.all(d[:, 4] == 3)


# --------------------------------------------------------------------------- P3 sphere
def test_sphere_impact_parameter(orc):
    grid = grid64()
    W = H = 24
    cam = cam_down(W=W, H=H, extent=0.9)
    h = 0.15625
    R, c = 20.0, 32.5
    rho0, kappa = 0.8, 4.0
    ball = lambda u, ctx: rho0 if (u[0] - c) ** 2 + (u[1] - c) ** 2 + (u[2] - c) ** 2 < R * R else 0.0
    r = orc.guiding_map(grid, None, cam, FRONT_DOWN, I.LIGHTS_EXPLICIT, I.Medium(kappa, 1.0, 0.0), march(h),
                        density_fn=ball)
    s = kappa * rho0 * h
    zs = 128.5 - 10.0 * np.arange(1, 14)
    checked = 0
    for q in range(W * H):
        px, py = q % W, q // W
        ux, uy = pixel_index_coords(cam, grid, px, py)
        b2 = (ux - c) ** 2 + (uy - c) ** 2
        d2 = (zs - c) ** 2
        if np.min(np.abs(d2 + b2 - R * R)) < 1e-2:
            continue                                     # sample on the sphere boundary: skip
        k = int(np.sum(d2 + b2 < R * R))
        assert r["rgbt"][q, 3] == pytest.approx(math.exp(-s * k), rel=1e-13)
        assert r["rgbt"][q, 0] == pytest.approx(slab_closed_form(s, k, I.EXP, 1.0, 1 / FOUR_PI, h), rel=1e-12, abs=1e-300)
        checked += 1
    assert checked > W * H * 0.9
    # a hole in the middle is visible: centre pixels see 4 samples, corners none
    assert r["rgbt"][:, 3].min() == pytest.approx(math.exp(-4 * s), rel=1e-12)


# --------------------------------------------------------------------------- P4 constant grid, apron
def test_constant_grid_apron_profile(orc):
    n, nz = 64, 60
    grid = grid64(n, nz)
    vals = np.full((nz, n, n), 0.25, np.float32)
    W = H = 20
    cam = cam_down(W=W, H=H, z=2.03125, extent=1.1)   # B_z = 130.5: samples at 60.5, 50.5, ..., 0.5
    h, kappa = 0.15625, 3.0
    r = orc.guiding_map(grid, vals, cam, FRONT_DOWN, I.LIGHTS_EXPLICIT, I.Medium(kappa, 1.0, 0.0), march(h))
    zs = 130.5 - 10.0 * np.arange(1, 15)
    zfac = np.clip(np.minimum(np.minimum(zs, nz + 1 - zs), 1.0), 0.0, None)   # apron ramps
    assert zfac[6] == 0.5 and zfac[12] == 0.5 and np.all(zfac[7:12] == 1.0) and not zfac[:6].any()
    ramp = lambda u, m: max(0.0, min(1.0, u, m + 1 - u))
    for q in range(W * H):
        px, py = q % W, q // W
        ux, uy = pixel_index_coords(cam, grid, px, py)
        rho = 0.25 * ramp(ux, n) * ramp(uy, n) * zfac
        sig = kappa * rho * h
        tau = np.cumsum(sig)
        Tprev = np.concatenate([[1.0], np.exp(-tau[:-1])])
        L = np.sum(Tprev * (1 - np.exp(-sig)) * Tprev) / FOUR_PI   # front light retraces: T^front_n = T_{n-1}
        assert r["rgbt"][q, 3] == pytest.approx(math.exp(-tau[-1]), rel=2e-6)
        assert r["rgbt"][q, 0] == pytest.approx(L, rel=2e-6, abs=1e-300)
        # continuum: optical depth through the grid along z is kappa * rho_xy * nz dx (exact for the ramp profile)


# --------------------------------------------------------------------------- P5, P6, P7
def test_conservation_exp(orc):
    """With h_l beyond the box every light march is empty (T^l = 1) and
    L_c = sum_l rgb_l P_l * alpha (1 - T)  (telescoping of A_n = alpha (T_{n-1} - T_n))."""
    w = I.make_workload("C1")
    med = I.Medium(32.0, 0.8, 0.4)
    m = w.march
    m2 = I.March(**{**m.__dict__, "light_step": 1e6, "t_min": 0.0})
    lights = [I.Light((0, 0, 0), (1.0, 0.5, 0.25)), I.Light((0, 0, 0), (0.3, 0.3, 0.3)),
              I.Light((0, 0, 0), (0.0, 1.0, 2.0))]
    r = orc.guiding_map(w.grid, w.volume(0), w.cameras[0], lights, I.LIGHTS_GUIDE, med, m2)
    fc = orc.frame_constants(w.grid, w.cameras[0], lights, I.LIGHTS_GUIDE, med, m2)
    T = r["rgbt"][:, 3]
    for c in range(3):
        wsum = sum(float(np.float32(lights[l].rgb[c])) * fc["P64"][l] for l in range(3))
        alpha = float(np.float32(0.8))
        np.testing.assert_allclose(r["rgbt"][:, c], wsum * alpha * (1 - T), rtol=1e-11, atol=1e-16)
    assert np.all(r["debug"][:, 5] == 0)
    assert np.any(T < 0.5)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_bounds_and_monotone_T(orc, cfg):
    w = I.make_workload(cfg, frames=[0])
    pix = np.arange(0, w.width * w.height, 7)
    r = orc.run_workload_frame(w, 0, pixels=pix)
    fc = orc.frame_constants(w.grid, w.cameras[0], w.lights[0], w.light_mode, w.medium, w.march)
    T = r["rgbt"][:, 3]
    assert np.all(T > 0) and np.all(T <= 1)
    for c in range(3):
        bound = w.medium.albedo * (1 - T) * sum(w.lights[0][l].rgb[c] * fc["P64"][l] for l in range(w.n_lights))
        assert np.all(r["rgbt"][:, c] >= 0)
        assert np.all(r["rgbt"][:, c] <= bound * (1 + 1e-12) + 1e-300)
    # T_N is non-increasing in N (Alg. 1 "for n <- 1 to N")
    prev = np.ones(len(pix))
    for N in range(1, 26, 3):
        mN = I.March(**{**w.march.__dict__, "max_steps": N})
        rN = orc.guiding_map(w.grid, w.volume(0), w.cameras[0], w.lights[0], w.light_mode, w.medium, mN,
                             frame_id=w.frame_ids[0], pixels=pix)
        assert np.all(rN["rgbt"][:, 3] <= prev + 1e-15)
        prev = rN["rgbt"][:, 3]


def test_linearity_in_light_radiance_and_density_scale(orc):
    w = I.make_workload("C1", single_light=True)
    g, v, cam, m = w.grid, w.volume(0), w.cameras[0], w.march
    la = I.Light(I._f32t(I._unit((0.3, -0.5, 0.8))), (1.0, 0.0, 0.5))
    lb = I.Light(I._f32t(I._unit((-0.7, 0.2, 0.1))), (0.25, 2.0, 0.0))
    pix = np.arange(0, 128 * 128, 5)
    ra = orc.guiding_map(g, v, cam, [la], 0, w.medium, m, pixels=pix)
    rb = orc.guiding_map(g, v, cam, [lb], 0, w.medium, m, pixels=pix)
    rab = orc.guiding_map(g, v, cam, [la, lb], 0, w.medium, m, pixels=pix)
    np.testing.assert_allclose(rab["rgbt"][:, :3], ra["rgbt"][:, :3] + rb["rgbt"][:, :3], rtol=1e-12, atol=1e-18)
    l2 = I.Light(la.to_light, (2.0, 0.0, 1.0))
    r2 = orc.guiding_map(g, v, cam, [l2], 0, w.medium, m, pixels=pix)
    np.testing.assert_allclose(r2["rgbt"][:, :3], 2 * ra["rgbt"][:, :3], rtol=1e-14, atol=1e-18)
    # sigma_t = kappa rho: doubling rho (exact in fp32) and halving kappa changes nothing
    rs = orc.guiding_map(g, v * np.float32(2), cam, [la], 0, I.Medium(16.0, 1.0, 0.0), m, pixels=pix)
    np.testing.assert_allclose(rs["rgbt"], ra["rgbt"], rtol=1e-13, atol=1e-18)
    assert np.array_equal(rs["depth"], ra["depth"])


# --------------------------------------------------------------------------- P8 symmetry
def test_mirror_symmetry_side_lights(orc):
    grid = grid64()
    W = H = 16
    cam = cam_down(W=W, H=H, extent=1.0)
    c = 32.5
    blob = lambda u, ctx: max(0.0, 1.0 - math.sqrt((u[0] - c) ** 2 + (u[1] - c) ** 2 + (u[2] - c) ** 2) / 22.0) ** 2
    med = I.Medium(6.0, 1.0, 0.3)
    rp = orc.guiding_map(grid, None, cam, [I.Light((1.0, 0.0, 0.0), (1, 1, 1))], 0, med, march(0.15625), density_fn=blob)
    rm = orc.guiding_map(grid, None, cam, [I.Light((-1.0, 0.0, 0.0), (1, 1, 1))], 0, med, march(0.15625), density_fn=blob)
    Lp = rp["rgbt"][:, 0].reshape(H, W)
    Lm = rm["rgbt"][:, 0].reshape(H, W)
    assert Lp.max() > 1e-3
    np.testing.assert_allclose(Lp, Lm[:, ::-1], rtol=1e-5, atol=1e-9)
    assert not np.allclose(Lp, Lp[:, ::-1], rtol=1e-3)       # each light alone is asymmetric
    # the guide set (axis +y -> side lights along -x/+x) gives a self-mirrored image
    rg = orc.guiding_map(grid, None, cam, I.guide_lights(), I.LIGHTS_GUIDE, med,
                         march(0.15625, guide_axis=(0.0, 1.0, 0.0)), density_fn=blob)
    Lg = rg["rgbt"][:, 0].reshape(H, W)
    np.testing.assert_allclose(Lg, Lg[:, ::-1], rtol=1e-5, atol=1e-9)


def test_rotation_about_view_axis(orc):
    """Rotating density, camera up vector and light by 90 deg about the view axis
    rotates the image by 90 deg (geometry of C3/C8 is frame-consistent)."""
    grid = grid64()
    W = H = 16
    c = 32.5
    rho = lambda x, y, z: max(0.0, 1.0 - math.sqrt(((x - c) / 1.5) ** 2 + (y - c - 4) ** 2 + (z - c) ** 2) / 18.0)
    d0 = lambda u, ctx: rho(u[0], u[1], u[2])
    d1 = lambda u, ctx: rho(u[1], 2 * c - u[0], u[2])    # rotated by +90 deg about z
    med = I.Medium(5.0, 1.0, 0.0)
    cam0 = cam_down(W=W, H=H, extent=1.0)
    cam1 = I.Camera(I.ORTHO, (0.5, 0.5, 2.0), (0.0, 0.0, -1.0), (-1.0, 0.0, 0.0), 1.0, W, H)
    l0 = [I.Light((0.6, 0.0, 0.8), (1, 1, 1))]
    l1 = [I.Light((0.0, 0.6, 0.8), (1, 1, 1))]
    r0 = orc.guiding_map(grid, None, cam0, l0, 0, med, march(0.15625), density_fn=d0)
    r1 = orc.guiding_map(grid, None, cam1, l1, 0, med, march(0.15625), density_fn=d1)
    np.testing.assert_allclose(r0["rgbt"].reshape(H, W, 4), r1["rgbt"].reshape(H, W, 4), rtol=2e-5, atol=1e-9)


# --------------------------------------------------------------------------- P9 opaque voxel
def test_single_opaque_voxel_depth(orc):
    """an opaque voxel on a pixel ray at distance d gives D in [d-h, d+h], T <= 1e-6."""
    n = 64
    grid = grid64(n)
    W = H = 64
    cam = cam_down(W=W, H=H, z=2.0, extent=1.0)        # pixel (px,py) ray passes x=(px+.5)/64, y=(63-py+.5)/64
    h = 0.15625
    i, j = 40, 23
    q = (63 - j) * W + i
    for jit, ks in ((0, [28]), (1, list(range(20, 40)))):
        vals = np.zeros((n, n, n), np.float32)
        for k in ks:
            vals[k, j, i] = 1e6
        r = orc.guiding_map(grid, vals, cam, FRONT_DOWN, 0, I.Medium(1.0, 1.0, 0.0),
                            march(h, jitter=jit, depth_tau=0.5), frame_id=3)
        d = 2.0 - (max(ks) + 0.5) / n                   # image plane z = 2 down to the top voxel centre
        assert d - 1.0 / n <= r["depth"][q] <= d + h
        assert r["rgbt"][q, 3] <= 1e-6
        assert 0 < np.sum(r["depth"] > 0) <= 9          # only rays within one voxel see it


# --------------------------------------------------------------------------- P10 clip = brute force
@pytest.mark.parametrize("persp", [False, True])
def test_clip_equals_unclipped_loop(orc, persp):
    w = I.make_workload("C1", perspective=persp)
    r1 = orc.run_workload_frame(w, 0)
    r2 = orc.run_workload_frame(w, 0, no_clip_n=400)
    for key in ("rgbt", "depth", "debug"):
        assert np.array_equal(r1[key], r2[key])
    assert r1["debug"][:, 0].max() > 0


# --------------------------------------------------------------------------- P11 convergence
def _continuum_T(vals, O, D, t_max, n=20001):
    t = np.linspace(0.0, t_max, n)
    u = O[None, :] + t[:, None] * D[None, :]
    rho = _trilinear_np(vals, u)
    # Simpson on a fine grid; the trilinear field is piecewise cubic along the line
    wts = np.ones(n); wts[1:-1:2] = 4; wts[2:-1:2] = 2
    return np.sum(wts * rho) * (t[1] - t[0]) / 3.0


def test_fine_step_convergence_front_light(orc):
    """As h -> 0 the EXP march converges to the continuum of eq:approx with the
    front light only: T = exp(-tau), L = P alpha (1 - T^2)/2 (exact identity)."""
    n = 8
    rng = np.random.default_rng(5)
    vals = (rng.random((n, n, n)) ** 2).astype(np.float32)
    grid = I.Grid(n, n, n, (0.0, 0.0, 0.0), float(np.float32(1.0 / n)))
    W = H = 6
    cam = cam_down(W=W, H=H, z=2.0, extent=0.7)
    kappa = 6.0
    med = I.Medium(kappa, 1.0, 0.0)
    # continuum along each pixel ray (index space: D = (0,0,-n) per world unit)
    cont_T, cont_L = [], []
    for q in range(W * H):
        ux, uy = pixel_index_coords(cam, grid, q % W, q // W)
        O = np.array([ux, uy, 2.0 * n + 0.5])
        D = np.array([0.0, 0.0, -float(n)])
        tau = kappa * _continuum_T(vals, O, D, 2.1) / 1.0
        cont_T.append(math.exp(-tau))
        cont_L.append((1 - math.exp(-2 * tau)) / 2 / FOUR_PI)
    cont_T, cont_L = np.array(cont_T), np.array(cont_L)
    errs_T, errs_L = [], []
    for mult in (2.0, 1.0, 0.5, 0.25, 0.125, 1.0 / 32):
        h = float(np.float32(mult / n))                 # h = mult * dx (world units)
        r = orc.guiding_map(grid, vals, cam, FRONT_DOWN, 0, med, march(h))
        errs_T.append(np.mean(np.abs(r["rgbt"][:, 3] - cont_T)))
        errs_L.append(np.mean(np.abs(r["rgbt"][:, 0] - cont_L)))
    assert all(b < a for a, b in zip(errs_T[2:], errs_T[3:])), errs_T
    assert all(b < a for a, b in zip(errs_L[2:], errs_L[3:])), errs_L
    assert errs_T[-1] < 2e-3 and errs_L[-1] < 2e-3


# --------------------------------------------------------------------------- ray geometry via the density hook
def test_sample_positions_lie_on_pixel_rays(orc):
    """The density callback sees every sample position the oracle evaluates: primary
    samples are t_n = delta + n h along the pixel ray of the camera model, light samples
    are spaced h_l along the light direction from their primary sample."""
    grid = grid64(32)
    W, H = 7, 5
    for proj in (I.ORTHO, I.PERSP):
        cam = I.Camera(proj, (0.2, -1.1, 0.9), I._f32t(I._unit((0.3, 1.6, -0.4))), (0.0, 0.0, 1.0),
                       1.3 if proj == I.ORTHO else 2 * math.tan(math.radians(35)), W, H)
        # independent fp64 camera basis
        f = np.array(cam.forward, np.float64); f /= np.linalg.norm(f)
        rr = np.cross(f, cam.up); rr /= np.linalg.norm(rr)
        uu = np.cross(rr, f)
        seen = []
        n_rays_hit = 0
        hook = lambda u, ctx: (seen.append((u[0], u[1], u[2])), 0.3)[1]
        h = float(np.float32(10.0 / 32))
        lt = I.Light(I._f32t(I._unit((0.1, -0.2, 0.97))), (1, 1, 1))
        for q in range(W * H):
            px, py = q % W, q // W
            seen.clear()
            m = march(h, jitter=1, seed=99, t_min=0.0)
            orc.guiding_map(grid, None, cam, [lt], 0, I.Medium(0.01, 1.0, 0.0), m, frame_id=2, pixels=[q],
                            density_fn=hook)
            sx = 2 * (px + .5) / W - 1
            sy = 1 - 2 * (py + .5) / H
            ay = cam.extent / 2
            ax = ay * W / H
            if proj == I.ORTHO:
                o = np.array(cam.position) + sx * ax * rr + sy * ay * uu
                d = f
            else:
                o = np.array(cam.position, np.float64)
                d = f + sx * ax * rr + sy * ay * uu
                d /= np.linalg.norm(d)
            if not seen:
                continue
            n_rays_hit += 1
            pts = (np.array(seen) - 0.5) / 32.0          # back to world space
            delta = orc.jitter_delta(m, 2, q)
            # primary samples are those on the ray
            tt = (pts - o) @ d
            off = np.linalg.norm(pts - o - tt[:, None] * d[None, :], axis=1)
            prim = off < 1e-4
            steps = (tt[prim] - delta) / h
            np.testing.assert_allclose(steps, np.round(steps), atol=1e-4)
            assert np.all(np.diff(np.round(steps)) == 1)
            # light samples: spaced h along the light direction from the preceding primary sample
            ld = np.array(lt.to_light, np.float64); ld /= np.linalg.norm(ld)
            idx = np.where(prim)[0]
            for a, b in zip(idx, list(idx[1:]) + [len(pts)]):
                seg = pts[a + 1:b] - pts[a]
                if len(seg):
                    jj = seg @ ld / h
                    np.testing.assert_allclose(jj, np.arange(1, len(seg) + 1), atol=1e-4)
                    nxt = pts[a] + (len(seg) + 1) * h * ld       # the first sample past the exit
                    un = nxt * 32 + 0.5
                    assert np.any((un <= 1e-3) | (un >= 33 - 1e-3))
        assert n_rays_hit >= 8


# --------------------------------------------------------------------------- early termination
def test_early_termination_rule(orc):
    w = I.make_workload("C2", frames=[0], kappa=128.0)
    pix = np.arange(0, 512 * 512, 97)
    m = w.march
    r = orc.run_workload_frame(w, 0, pixels=pix)
    d = r["debug"]
    term = d[:, 3] < d[:, 1]
    assert term.sum() > 10
    assert np.all(r["rgbt"][term, 3] < m.t_min)
    # without the rule, T at the termination step is the same and later steps only lower it
    m0 = I.March(**{**m.__dict__, "t_min": 0.0})
    r0 = orc.guiding_map(w.grid, w.volume(0), w.cameras[0], w.lights[0], w.light_mode, w.medium, m0,
                         frame_id=w.frame_ids[0], pixels=pix)
    assert np.all(r0["rgbt"][term, 3] <= r["rgbt"][term, 3])
    assert np.all(r0["debug"][:, 3] == r0["debug"][:, 1])
    # forcing n_term to the natural value reproduces the run bit for bit
    rf = orc.guiding_map(w.grid, w.volume(0), w.cameras[0], w.lights[0], w.light_mode, w.medium, m0,
                         frame_id=w.frame_ids[0], pixels=pix,
                         forced_term=np.where(term, d[:, 3], -1).astype(np.int32))
    assert np.array_equal(rf["rgbt"][term], r["rgbt"][term])


def test_early_termination_is_the_first_crossing(orc):
    """C11: n_term is the FIRST step whose T_n (fp32
    decision) falls below T_min.  T_n is taken from runs with the rule switched off
    (t_min = 0) and capped at N (Alg. 1's step count input): at N = n_term
    T < T_min, at N = n_term - 1 still T >= T_min; pixels that never terminate keep
    T >= T_min at n_hi.  An oracle that stops one occupied step late (or early) fails."""
    w = I.make_workload("C2", frames=[0], kappa=128.0)
    pix = np.arange(0, 512 * 512, 53)
    m = w.march
    r = orc.run_workload_frame(w, 0, pixels=pix)
    d = r["debug"].astype(np.int64)
    term = (d[:, 3] > 0) & (d[:, 3] < d[:, 1])
    assert term.sum() > 50
    assert np.all(r["rgbt"][~term & (d[:, 0] > 0), 3].astype(np.float32) >= np.float32(m.t_min))
    T_at = {}
    for N in sorted(set(d[term, 3].tolist()) | set((d[term, 3] - 1).tolist())):
        sel = term & ((d[:, 3] == N) | (d[:, 3] - 1 == N))
        mN = I.March(**{**m.__dict__, "t_min": 0.0, "max_steps": int(N)})
        rN = orc.guiding_map(w.grid, w.volume(0), w.cameras[0], w.lights[0], w.light_mode, w.medium, mN,
                             frame_id=w.frame_ids[0], pixels=pix[sel])
        for p, t in zip(pix[sel], rN["rgbt"][:, 3]):
            T_at[(int(p), int(N))] = np.float32(t)
    for p, nt in zip(pix[term], d[term, 3]):
        assert T_at[(int(p), int(nt))] < np.float32(m.t_min), (p, nt)
        assert T_at[(int(p), int(nt) - 1)] >= np.float32(m.t_min), (p, nt)
        # and the terminated run reports exactly T_{n_term}
    assert np.array_equal(r["rgbt"][term, 3].astype(np.float32),
                          np.array([T_at[(int(p), int(nt))] for p, nt in zip(pix[term], d[term, 3])]))


def test_guide_axis_fallback_closed_form(orc):
    """Ledger #8 ("omega x z"): when omega is parallel to the guide axis,
    omega x z vanishes and the side lights fall back to +-normalize(omega x x_hat).  A camera
    looking straight down (forward -z, omega = +z) with axis z gives omega x x_hat =
    (0,0,1) x (1,0,0) = (0,1,0): top = +y_hat, bottom = -y_hat, front = +z_hat (closed form)."""
    g = grid64(32)
    med = I.Medium(32.0, 1.0, 0.0)
    guide = I.guide_lights()
    inv = np.float32(1.0 / np.float64(g.voxel_width))
    fc = orc.frame_constants(g, cam_down(), guide, I.LIGHTS_GUIDE, med, march(10.0 / 32))
    np.testing.assert_array_equal(fc["Ln"], np.array([[0, 0, 1], [0, 1, 0], [0, -1, 0]], np.float32))
    np.testing.assert_array_equal(fc["Lg"], np.array([[0, 0, inv], [0, inv, 0], [0, -inv, 0]], np.float32))
    # omega = -z (camera looking up): (0,0,-1) x (1,0,0) = (0,-1,0)
    cam_up = I.Camera(I.ORTHO, (0.5, 0.5, -1.0), (0.0, 0.0, 1.0), (0.0, 1.0, 0.0), 0.9, 32, 32)
    fc = orc.frame_constants(g, cam_up, guide, I.LIGHTS_GUIDE, med, march(10.0 / 32))
    np.testing.assert_array_equal(fc["Ln"], np.array([[0, 0, -1], [0, -1, 0], [0, 1, 0]], np.float32))
    # rendered consequence: with a blob off-centre in +y (and centred in x) the guide set's
    # image equals front + explicit lights along the closed-form directions +-y (additivity
    # over lights, P7) -- and differs from the +-x pair a wrong fallback would pick
    vals = np.zeros((32, 32, 32), np.float32)
    vals[10:22, 21:27, 8:24] = 0.7
    m = march(1.0 / 32)

    def explicit(d):
        return orc.guiding_map(g, vals, cam_down(), [I.Light(d, (1.0, 1.0, 1.0))], I.LIGHTS_EXPLICIT, med,
                               m)["rgbt"][:, 0]

    gm = orc.guiding_map(g, vals, cam_down(), guide, I.LIGHTS_GUIDE, med, m)["rgbt"][:, 0]
    front = explicit((0.0, 0.0, 1.0))
    np.testing.assert_allclose(gm, front + explicit((0.0, 1.0, 0.0)) + explicit((0.0, -1.0, 0.0)),
                               rtol=1e-12, atol=1e-15)
    wrong = front + explicit((1.0, 0.0, 0.0)) + explicit((-1.0, 0.0, 0.0))
    assert np.abs(gm - wrong).max() > 1e-3 * np.abs(gm).max()


def test_depth_threshold_is_strict(orc):
    """C6 / Alg. 1 line "if D = 0 and sigma_n > tau": strict.  A constant grid
    with sigma_s exactly tau on its plateau (rho 0.5, kappa 2, alpha 1: sigma_s = 1.0 exactly,
    P13's exact interior) never hits at tau = 1.0, and hits at the first plateau sample once tau is
    one fp32 ulp lower -- there D equals the t of the first sample with rho = 0.5 exactly."""
    g = grid64(16)
    vals = np.full((16, 16, 16), 0.5, np.float32)
    cam = cam_down(W=8, H=8, extent=0.5)
    med = I.Medium(2.0, 1.0, 0.0)
    r = orc.guiding_map(g, vals, cam, FRONT_DOWN, I.LIGHTS_EXPLICIT, med, march(1.0 / 64, depth_tau=1.0))
    assert np.all(r["depth"] == 0.0) and np.all(r["debug"][:, 2] == 0)
    tau = float(np.nextafter(np.float32(1.0), np.float32(0.0)))
    r = orc.guiding_map(g, vals, cam, FRONT_DOWN, I.LIGHTS_EXPLICIT, med, march(1.0 / 64, depth_tau=tau))
    assert np.all(r["depth"] > 0.0)
    # the first hit: sample n at z = 2 - n/64 has padded index u_z = 16 (2 - n/64) + 1/2, and the
    # trilinear value is exactly 0.5 once u_z <= 16 (at u_z = 16 the weight of the apron corner is
    # 0): 16 (2 - n/64) + 1/2 <= 16  <=>  n >= 66, so D = 66 h = 1.03125 for every pixel
    assert np.all(r["debug"][:, 2] == 66) and np.all(r["depth"] == np.float32(66 / 64))


def test_golden_hash_table_is_current(orc):
    """tests/golden/jitter_hash.txt was written by tests/golden/make_golden.py from the oracle."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "jitter_hash.txt")
    rows = [l.split() for l in open(path) if not l.startswith("#")]
    assert len(rows) == 64
    for p, hx in rows:
        assert orc.jitter_hash(0x26040374, 7, int(p)) == int(hx, 16)
