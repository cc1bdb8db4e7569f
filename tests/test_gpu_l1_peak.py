"""The hardware L1/TEX ceiling microbenchmark (nsl_bench_l1_peak) loads what it
reports: on a buffer of ones every load adds 8, so each thread's sum is reps x 16 x 8."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_l1_peak_loads_every_element():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    import paper_2604_03748_b200 as nsl
    reps = 4
    off = torch.randint(0, 1000, (16, 32), dtype=torch.int32, device="cuda")
    buf = torch.ones((1000 + 77 + 1) * 8, dtype=torch.float32, device="cuda")
    sink = torch.full((148 * 8 * 256,), -1.0, dtype=torch.float32, device="cuda")
    nbytes = nsl.bench_l1_peak(buf, off, stride=13, span=77, waves=1, reps=reps, sink=sink)
    torch.cuda.synchronize()
    threads = nbytes // (reps * 16 * 32)
    assert nbytes == threads * reps * 16 * 32 and threads % (148 * 256) == 0
    assert np.all(sink[:threads].cpu().numpy() == np.float32(reps * 16 * 8))
    with pytest.raises(nsl.NslError):          # a span beyond the buffer is refused, not read
        nsl.bench_l1_peak(buf, off, stride=13, span=10 ** 6, waves=1, reps=reps, sink=sink)
