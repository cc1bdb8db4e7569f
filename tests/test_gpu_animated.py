"""nsl_guiding_map_animated (rows a1 + a9, C4: a fresh density grid per frame, layouts of the
next chunk built on a side stream while the current chunk marches): bitwise equal to per-frame
uploads + one batch call, values within the bar against the oracle, invalid densities counted."""
from dataclasses import replace

import numpy as np
import pytest

import nsl_inputs as I
from parity import compare_frame, fast_decisions

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    import paper_2604_03748_b200 as nsl
    nsl.lib()
    return nsl


FRAMES = [0, 1, 2, 3, 4, 120, 239]


def _inputs(nsl, w, layout):
    import torch
    raw = [torch.from_numpy(w.volume(i)).cuda() for i in range(len(w.volume_specs))]
    dens = [raw[w.frame_vol[f]] for f in range(w.n_frames)]
    nb = nsl.volume_bytes(w.grid, layout)
    stor = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(w.n_frames)]
    return raw, dens, stor


def _animated(nsl, w, layout, chunk, check=False):
    import torch
    raw, dens, stor = _inputs(nsl, w, layout)
    rgbt, depth, _ = nsl.alloc_outputs(w.n_frames, w.height, w.width)
    n = nsl.guiding_map_animated(w.grid, dens, layout, stor, w.cameras, w.lights, w.light_mode, w.medium, w.march,
                                 w.frame_ids, rgbt, depth, chunk=chunk, check=check)
    torch.cuda.synchronize()
    return rgbt.cpu().numpy(), depth.cpu().numpy(), n


@pytest.mark.parametrize("layout,light_model", [(1, 0), (3, 0), (3, 1)])
def test_animated_equals_upload_plus_batch(nsl, layout, light_model):
    import torch
    w = I.make_workload("C4", frames=FRAMES)
    w = replace(w, march=replace(w.march, light_model=light_model))
    ref = nsl.run_workload(w, layout=layout)
    torch.cuda.synchronize()
    ref = (ref[0].cpu().numpy(), ref[1].cpu().numpy())
    for chunk in (0, 1, 3, 100):
        g, gd, _ = _animated(nsl, w, layout, chunk)
        assert np.array_equal(g, ref[0]) and np.array_equal(gd, ref[1]), chunk


def test_animated_parity_sampled(nsl):
    w = I.make_workload("C4", frames=FRAMES)
    g, gd, n = _animated(nsl, w, 3, 0, check=True)
    assert n == 0
    dbg = nsl.run_workload(w, layout=3, debug=True)
    dec = fast_decisions((g, gd), tuple(t.cpu().numpy() for t in dbg))
    pix = np.arange(0, w.height * w.width, 211)
    for f in (0, 5, 6):
        compare_frame(w, f, g[f], gd[f], None, pixels=pix, dec=dec[f])


def test_animated_counts_invalid_density(nsl):
    import torch
    w = I.make_workload("C4", frames=[0, 1, 2, 3])
    raw, dens, stor = _inputs(nsl, w, 3)
    bad = dens[2].clone()
    bad.view(-1)[12345] = float("nan")
    bad.view(-1)[777] = -1.0
    dens[2] = bad
    rgbt, depth, _ = nsl.alloc_outputs(w.n_frames, w.height, w.width)
    n = nsl.guiding_map_animated(w.grid, dens, 3, stor, w.cameras, w.lights, w.light_mode, w.medium, w.march,
                                 w.frame_ids, rgbt, depth, check=True)
    torch.cuda.synchronize()
    assert n == 2
