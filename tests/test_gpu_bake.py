"""GPU parity of the NEXT-1 six-way bake against the oracle:
same counter-based sample positions on both sides, so the estimator values are
compared element by element (|gpu - oracle| <= max(1e-4 |oracle|, 1e-5))."""
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


def bake_gpu(nsl, w, b, layout=1):
    import torch
    out = nsl.run_bake(w, b, layout=layout)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(w.n_frames, -1, 8)


def check(g, o, what=""):
    err = np.abs(g.astype(np.float64) - o)
    tol = np.maximum(1e-4 * np.abs(o), 1e-5)
    bad = err > tol
    assert not bad.any(), f"{what}: {int(bad.sum())} bad, worst gpu {g[bad][:3]} oracle {o[bad][:3]}"


def test_bake_lights_bitwise(nsl):
    for cfg in ("C1", "C2", "C3"):
        w = I.make_workload(cfg, frames=[0])
        a = nsl.debug_bake_lights(w.grid, w.cameras[0])
        b = oracle.bake_light_constants(w.grid, w.cameras[0])
        for x, y in zip(a, b):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


@pytest.mark.parametrize("persp", [False, True])
def test_bake_parity_C1(nsl, persp):
    w = I.make_workload("C1", perspective=persp)
    b = I.default_bake(64, spp=4)
    g = bake_gpu(nsl, w, b)[0]
    o = oracle.sixway_bake(w.grid, w.volume(0), w.cameras[0], w.medium, b, frame_id=w.frame_ids[0])["out"]
    check(g, o, "C1")
    assert o[:, [0, 1, 2, 4, 5, 6]].max() > 1e-3 and o[:, 3].min() < 0.5


def test_bake_parity_C2_subsampled_and_layouts(nsl):
    w = I.make_workload("C2", frames=[0, 17])
    b = I.default_bake(128, spp=2)
    pix = np.arange(0, 512 * 512, 61)
    ref = [oracle.sixway_bake(w.grid, w.volume(0), w.cameras[f], w.medium, b, frame_id=w.frame_ids[f],
                              pixels=pix)["out"] for f in range(2)]
    for layout in (0, 1, 3, 5, 6):
        g = bake_gpu(nsl, w, b, layout)
        for f in range(2):
            check(g[f][pix], ref[f], f"C2 f{f} layout {layout}")


def test_bake_random_tiny_cases_and_determinism(nsl):
    import torch
    rng = np.random.default_rng(77)
    for trial in range(12):
        n = int(rng.integers(5, 14))
        grid = I.Grid(n, n, n, (0.0, 0.0, 0.0), float(np.float32(1.0 / n)))
        vals = (rng.random((n, n, n)) * (rng.random((n, n, n)) < 0.5)).astype(np.float32)
        cam = I.orbit_camera(rng.uniform(0, 360), int(rng.integers(3, 17)), int(rng.integers(3, 17)),
                             elev_deg=rng.uniform(-50, 50), projection=int(rng.integers(0, 2)),
                             extent=float(rng.uniform(0.8, 2.0)))
        med = I.Medium(float(np.float32(rng.uniform(2, 60))), float(np.float32(rng.uniform(0.3, 1))),
                       float(np.float32(rng.uniform(-0.6, 0.6))))
        b = I.Bake(spp=int(rng.integers(1, 40)), step=float(np.float32(rng.uniform(0.3, 1.5) / n)),
                   light_step=float(np.float32(rng.uniform(0.5, 3.0) / n)), t_min=float(rng.choice([0.0, 1e-3])),
                   seed=int(rng.integers(0, 2 ** 62)))
        w = I.Workload(name="tiny", grid=grid, volume_specs=[("given", 0)], frame_vol=[0], cameras=[cam],
                       light_mode=0, lights=[[I.Light((1.0, 0.0, 0.0), (1, 1, 1))]], medium=med,
                       march=I.March(step=grid.voxel_width), frame_ids=[int(rng.integers(0, 99))], _cache={0: vals})
        g = bake_gpu(nsl, w, b)
        o = oracle.sixway_bake(grid, vals, cam, med, b, frame_id=w.frame_ids[0])["out"]
        check(g[0], o, f"trial {trial}")
        assert np.array_equal(g, bake_gpu(nsl, w, b))                  # bitwise deterministic


def test_bake_zero_volume(nsl):
    w = I.make_workload("C1")
    w._cache[0] = np.zeros_like(w.volume(0))
    g = bake_gpu(nsl, w, I.default_bake(64, spp=3))[0]
    assert np.all(g[:, [0, 1, 2, 4, 5, 6, 7]] == 0.0) and np.all(g[:, 3] == 1.0)
