"""Writes tests/golden/*.txt.  Calls ONLY oracle/ (DESIGN.md §3): stored values
are the oracle's, never the CUDA path's.

jitter_hash.txt — DESIGN.md C4 hash chain for seed 0x26040374, frame 7,
pixels 0..63 (pin P14: cross-checked against the GPU's independent
implementation in tests/test_gpu_parity.py).  The chain's building block is
pinned separately to the published MurmurHash3 fmix32 values
(tests/test_oracle_pins.py::test_fmix32_published_values).
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

SEED, FRAME = 0x26040374, 7


def main():
    with open(os.path.join(HERE, "jitter_hash.txt"), "w") as f:
        f.write("# DESIGN.md C4 jitter hash, seed=0x26040374 frame=7, pixel index -> h32 (hex)\n")
        for p in range(64):
            f.write("%d %08x\n" % (p, oracle.jitter_hash(SEED, FRAME, p)))


if __name__ == "__main__":
    main()
