"""Run A/B variants built by scripts/ab_local.sh on the GPU, interleaved:
    python scripts/ab_run.py NAME [NAME ...] [--reps 3] [--bench-args "--config C2"]
prints one line per (rep, variant): step ms, march ms, clocks."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
p = argparse.ArgumentParser()
p.add_argument("names", nargs="+")
p.add_argument("--reps", type=int, default=3)
p.add_argument("--steps", type=int, default=100)
p.add_argument("--bench-args", default="")
a = p.parse_args()
res = {n: [] for n in a.names}
for rep in range(a.reps):
    for n in a.names:
        env = dict(os.environ, NSL_LIB=os.path.join(ROOT, "abl", f"libnsl_{n}.so"))
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(a.steps), "--warmup", "3", "--no-e2e",
               "--no-cpu-baseline", "--no-sampler-ceiling", *a.bench_args.split()]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            res[n].append(d["march_ms_per_step"])
            print(f"{n:16s} rep{rep} step={d['ms_per_step']:.4f} march={d['march_ms_per_step']:.4f} "
                  f"clk={d['clocks']['sm_mhz']} {a.bench_args}", flush=True)
        except Exception:
            print(n, "FAILED", r.stdout[-300:], r.stderr[-1500:], flush=True)
for n, v in res.items():
    if v:
        print(f"SUMMARY {n:16s} march min {min(v):.4f} median {sorted(v)[len(v) // 2]:.4f} {a.bench_args}")
