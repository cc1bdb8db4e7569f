"""The sampler microbenchmark (nsl_bench_l1_gather, SURVEY §8(d) denominators) takes the samples
it reports: on a constant grid every in-support trilinear sample is the constant (C1, P4), so
each thread's sum is exactly reps x 16 x c."""
import numpy as np
import pytest

import nsl_inputs as I

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layout", [0, 1, 2, 3, 4])
def test_l1_gather_constant_grid(layout):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    import paper_2604_03748_b200 as nsl
    n, c, reps = 16, 0.5, 8
    dens = torch.full((n, n, n), c, dtype=torch.float32, device="cuda")
    vol = nsl.Volume(I.Grid(n, n, n, (0.0, 0.0, 0.0), 1.0 / n), dens, layout)
    sink = torch.full((148 * 16 * 128,), -1.0, dtype=torch.float32, device="cuda")
    samples = nsl.bench_l1_gather(vol, sink, waves=1, reps=reps)
    torch.cuda.synchronize()
    threads = samples // (reps * 16)
    assert samples == threads * reps * 16 and threads % (148 * 128) == 0
    got = sink[:threads].cpu().numpy()
    assert np.all(got == np.float32(reps * 16 * c))
