"""Pins of the NEXT-4 transmittance-volume oracle (V2-V6), checked against
things other than itself: the canonical light march C8 (pinned in test_oracle_pins.py), a
numpy closed form on the raw grid for an axis-aligned light, the mirror lattice built
independently, an analytic line integral under grid refinement, and the canonical
guiding map's bookkeeping."""
import math

import numpy as np
import pytest

import nsl_inputs as I
import oracle


@pytest.fixture(scope="module")
def c1():
    w = I.make_workload("C1")
    fc = oracle.frame_constants(w.grid, w.cameras[0], w.lights[0], w.light_mode, w.medium, w.march)
    hl = w.march.light_step if w.march.light_step > 0 else w.march.step
    return w, fc, np.float32(hl)


def test_lattice_is_orthonormal_and_covers_the_support(c1):
    w, fc, hl = c1
    for Lg in fc["Lg"][1:]:
        lat = oracle.tv_lattice(w.grid, Lg, hl)
        E = np.array([lat.e1[:], lat.e2[:], lat.dhat[:]])
        np.testing.assert_allclose(E @ E.T, np.eye(3), atol=1e-12)
        np.testing.assert_allclose(np.array(lat.d[:]), lat.ell * np.array(lat.dhat[:]), rtol=1e-14)
        np.testing.assert_allclose(np.array(lat.d[:]), float(hl) * Lg.astype(np.float64), rtol=1e-14)
        rng = np.random.default_rng(0)
        n = np.array([w.grid.nx + 1, w.grid.ny + 1, w.grid.nz + 1], np.float64)
        U = rng.random((2000, 3)) * n
        a = U @ np.array(lat.e1[:]) - lat.a0
        b = U @ np.array(lat.e2[:]) - lat.b0
        k = U @ np.array(lat.dhat[:]) / lat.ell - lat.k0
        assert a.min() >= 1 and a.max() <= lat.A - 2
        assert b.min() >= 1 and b.max() <= lat.B - 2
        assert k.min() >= 1 and k.max() <= lat.K - 2


def test_lattice_points_equal_the_canonical_light_march(c1):
    """V4: at a lattice point, tau+ is C8's optical depth from that point (same samples)."""
    w, fc, hl = c1
    vals = w.volume(0)
    kappa = float(np.float32(w.medium.extinction))
    Lg = fc["Lg"][1]
    lat = oracle.tv_lattice(w.grid, Lg, hl)
    tp, tm = oracle.tv_build(w.grid, vals, lat, float(hl), kappa)
    rng = np.random.default_rng(1)
    e1, e2, d = np.array(lat.e1[:]), np.array(lat.e2[:]), np.array(lat.d[:])
    checked = 0
    for _ in range(400):
        i, j, k = rng.integers(1, lat.A - 1), rng.integers(1, lat.B - 1), rng.integers(1, lat.K - 1)
        P = (lat.a0 + i) * e1 + (lat.b0 + j) * e2 + (lat.k0 + k) * d
        if not (np.all(P > 0.5) and np.all(P < np.array([w.grid.nx, w.grid.ny, w.grid.nz]) + 0.5)):
            continue
        U = P.astype(np.float32)
        ref = oracle.light_tau(w.grid, vals, U, Lg, float(hl), kappa)
        assert tp[j, k, i] == pytest.approx(ref, rel=2e-5, abs=1e-9)
        assert oracle.tv_lookup(lat, tp, U) == pytest.approx(ref, rel=2e-5, abs=1e-6)
        checked += 1
    assert checked > 100


def test_prefix_and_suffix_partition_each_line(c1):
    """V4 bookkeeping: tau+(k) + tau-(k) + kappa h rho(k) is the same line total for every k."""
    w, fc, hl = c1
    kappa = float(np.float32(w.medium.extinction))
    lat = oracle.tv_lattice(w.grid, fc["Lg"][1], hl)
    tp, tm = oracle.tv_build(w.grid, w.volume(0), lat, float(hl), kappa)
    own = np.zeros_like(tp)
    own[:, :-1, :] = tm[:, 1:, :] - tm[:, :-1, :]          # kappa h rho(k) from the prefix steps
    own[:, -1, :] = tp[:, -2, :] - tp[:, -1, :] if tp.shape[1] > 1 else 0.0
    tot = tp + tm + own
    np.testing.assert_allclose(tot, tot[:, :1, :].repeat(tot.shape[1], axis=1), rtol=1e-12, atol=1e-12)
    assert tot.max() > 1.0                                   # the lines do cross the smoke
    assert np.all(tm[:, 0, :] == 0.0) and np.all(tp[:, -1, :] == 0.0)


def test_mirror_lattice_gives_the_opposite_light(c1):
    """V5: the opposite light's own lattice holds the same lines, so its tau+ is tau- here."""
    w, fc, hl = c1
    kappa = float(np.float32(w.medium.extinction))
    vals = w.volume(0)
    L = fc["Lg"][1]
    la, lb = oracle.tv_lattice(w.grid, L, hl), oracle.tv_lattice(w.grid, -L, hl)
    tpa, tma = oracle.tv_build(w.grid, vals, la, float(hl), kappa)
    tpb, _ = oracle.tv_build(w.grid, vals, lb, float(hl), kappa)
    rng = np.random.default_rng(2)
    n = np.array([w.grid.nx, w.grid.ny, w.grid.nz], np.float64)
    for U in (rng.random((300, 3)) * n + 0.5).astype(np.float32):
        assert oracle.tv_lookup(lb, tpb, U) == pytest.approx(oracle.tv_lookup(la, tma, U), rel=1e-6, abs=1e-8)


def test_axis_aligned_light_closed_form():
    """L = +x with h_l = 2 voxels: lattice points are grid nodes, so tau+ is a plain sum of padded
    voxel values along x (numpy), and the lookup is numpy's trilinear interpolation of it."""
    n = 12
    g = I.Grid(n, n, n, (0.0, 0.0, 0.0), 1.0)
    rng = np.random.default_rng(5)
    vol = (rng.random((n, n, n)) * (rng.random((n, n, n)) < 0.6)).astype(np.float32)   # [z, y, x]
    kappa, hl = 3.0, 2.0
    Lg = np.array([1.0, 0.0, 0.0], np.float32)
    lat = oracle.tv_lattice(g, Lg, hl)
    assert np.allclose(lat.e1[:], (0, -1, 0)) and np.allclose(lat.e2[:], (0, 0, -1))
    tp, tm = oracle.tv_build(g, vol, lat, hl, kappa)
    pad = np.zeros((n + 2, n + 2, n + 2))
    pad[1:-1, 1:-1, 1:-1] = vol

    def rho_node(x, y, z):                  # C1 at an integer node inside the support, else 0
        if not (0 < x < n + 1 and 0 < y < n + 1 and 0 < z < n + 1):
            return 0.0
        return pad[z, y, x]

    ref = np.zeros_like(tp)
    for j in range(lat.B):
        for i in range(lat.A):
            y, z = -(lat.a0 + i), -(lat.b0 + j)
            line = [rho_node(2 * (lat.k0 + k), y, z) for k in range(lat.K)]
            suf = np.concatenate([np.cumsum(line[::-1])[::-1][1:], [0.0]])
            ref[j, :, i] = kappa * hl * suf
    np.testing.assert_allclose(tp, ref, rtol=1e-13, atol=1e-13)
    # lookup = trilinear in (a, b, k) = (-y, -z, x/2)
    for U in (rng.random((200, 3)) * (n + 1)).astype(np.float32):
        a, b, k = -float(U[1]) - lat.a0, -float(U[2]) - lat.b0, float(U[0]) / 2.0 - lat.k0
        i0, j0, k0 = int(math.floor(a)), int(math.floor(b)), int(math.floor(k))
        fa, fb, fk = a - i0, b - j0, k - k0
        v = 0.0
        for di in (0, 1):
            for dj in (0, 1):
                for dk in (0, 1):
                    wgt = (fa if di else 1 - fa) * (fb if dj else 1 - fb) * (fk if dk else 1 - fk)
                    v += wgt * ref[j0 + dj, k0 + dk, i0 + di]
        assert oracle.tv_lookup(lat, tp, U) == pytest.approx(v, rel=1e-12, abs=1e-12)


def test_converges_to_the_line_integral_under_refinement():
    """A smooth Gaussian blob (analytic density callback) and an oblique light: the lookup's
    optical depth approaches the exact line integral as the grid (and the light step) refine."""
    L = np.array([0.48, 0.36, 0.8])
    L /= np.linalg.norm(L)
    c0, s0 = np.array([0.5, 0.5, 0.5]), 0.12

    def rho_world(p):
        return math.exp(-float(np.sum((p - c0) ** 2)) / (2 * s0 * s0))

    pts = [np.array([0.45, 0.52, 0.40]), np.array([0.55, 0.47, 0.50]), np.array([0.50, 0.60, 0.45])]
    exact = []
    for p in pts:   # integral of rho along p + s L, s > 0 (fine midpoint rule in world units)
        ds = 1e-4
        s = np.arange(ds / 2, 1.8, ds)
        q = p[None, :] + s[:, None] * L[None, :]
        exact.append(np.sum(np.exp(-np.sum((q - c0) ** 2, axis=1) / (2 * s0 * s0))) * ds)
    errs = []
    for n in (16, 32, 64):
        dx = 1.0 / n
        g = I.Grid(n, n, n, (0.0, 0.0, 0.0), dx)

        def dens(u, _ctx, dx=dx):            # padded index position -> world: (u - 0.5) dx
            return rho_world(np.array([(u[0] - 0.5) * dx, (u[1] - 0.5) * dx, (u[2] - 0.5) * dx]))

        hl = dx                               # one voxel
        Lg = (L / dx).astype(np.float32)
        lat = oracle.tv_lattice(g, Lg, hl)
        tp, _ = oracle.tv_build(g, None, lat, hl, 1.0, density_fn=dens)
        e = 0.0
        for p, ex in zip(pts, exact):
            U = (p / dx + 0.5).astype(np.float32)
            e = max(e, abs(oracle.tv_lookup(lat, tp, U) - ex) / ex)
        errs.append(e)
    # first order (the right-endpoint rule of C8 misses ~h/2 of the line at its start):
    # the error at least ~halves per refinement
    assert errs[0] > 1.6 * errs[1] > 1.6 * 1.6 * errs[2], errs
    assert errs[2] < 0.08, errs


def test_zero_density_and_bookkeeping_unchanged(c1):
    """V1/V6: with light_model = 1 only T^l of the non-front lights changes: every debug counter,
    T, D and the front light's scattering equal the canonical run's; zero density gives T = 1."""
    import dataclasses
    w, fc, hl = c1
    base = oracle.run_workload_frame(w, 0)
    m_tv = dataclasses.replace(w.march, light_model=1)
    tv = oracle.guiding_map(w.grid, w.volume(0), w.cameras[0], w.lights[0], w.light_mode, w.medium, m_tv,
                            frame_id=w.frame_ids[0])
    assert np.array_equal(tv["debug"], base["debug"])
    assert np.array_equal(tv["depth"], base["depth"])
    assert np.array_equal(tv["rgbt"][:, 3], base["rgbt"][:, 3])
    diff = np.abs(tv["rgbt"][:, :3] - base["rgbt"][:, :3])
    scale = np.abs(base["rgbt"][:, :3]).max()
    assert diff.max() > 0.0                              # the side lights did change ...
    assert diff.max() < 0.1 * scale                      # ... by a discretisation-sized amount
    zero = oracle.guiding_map(w.grid, np.zeros_like(w.volume(0)), w.cameras[0], w.lights[0], w.light_mode,
                              w.medium, m_tv, frame_id=w.frame_ids[0])
    assert np.all(zero["rgbt"][:, 3] == 1.0) and np.all(zero["rgbt"][:, :3] == 0.0)
