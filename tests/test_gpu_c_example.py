"""The C example (examples/guiding_map_c.c) built with gcc and run on the GPU: plain C callers
get a guiding map through nsl_guiding_map_host and invalid input is rejected."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_c_example_runs(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    import paper_2604_03748_b200 as nsl
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = nsl.build()                      # the library in use (NSL_LIB may point at a build variant)
    libdir = os.path.dirname(lib)
    exe = tmp_path / "gm"
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", "guiding_map_c.c"), lib,
                           f"-Wl,-rpath,{libdir}", "-lm", "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("ok")
