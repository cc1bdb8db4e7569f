"""Mutation check of the oracle's pins: copy the repo to a scratch directory,
apply one plausible mistake at a time to oracle/nsl_oracle.c, rebuild the oracle there and run
the CPU pin suite (tests/test_oracle_pins.py); every mutant must make at least one pin fail.

    python scripts/oracle_mutants.py [--keep]
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTANTS = {
    # C11: terminate one occupied step late (after the first crossing, one more step)
    "C11 one step late": ("int terminated = 0;", "int terminated = 0; int crossed = 0;",
                          "if ((float)T < m->t_min) terminated = 1;",
                          "if (crossed) terminated = 1; if ((float)T < m->t_min) crossed = 1;"),
    # ledger #8: fall back to omega x y_hat instead of omega x x_hat
    "guide-axis fallback x->y": ("double xh[3] = {1.0, 0.0, 0.0};", "double xh[3] = {0.0, 1.0, 0.0};", None, None),
    # C7: opacity from T_n instead of T_{n-1} (EXP form)
    "C7 A_n uses T_n": ("if (m->opacity_form == 0) A = alpha * T_prev * (1.0 - exp(-s));",
                        "if (m->opacity_form == 0) A = alpha * T * (1.0 - exp(-s));", None, None),
    # C6: non-strict depth threshold
    # C8: left-endpoint light march (the sum starts at the sample y itself, j = 0)
    "C8 left endpoint": ("    uint32_t j = 1;\n    for (;; ++j) {\n        float s = (float)j * hl;",
                         "    uint32_t j = 1;\n    for (;; ++j) {\n        float s = (float)(j - 1) * hl;", None, None),
    # C3: image rows counted bottom-up (s_y sign)
    "C3 rows bottom-up": ("double ex = 2.0 / W, ey = -2.0 / H;", "double ex = 2.0 / W, ey = 2.0 / H;",
                          "double cx = 1.0 / W - 1.0, cy = 1.0 - 1.0 / H;",
                          "double cx = 1.0 / W - 1.0, cy = 1.0 / H - 1.0;"),
    # C10: phase angle with the wrong sign convention (front light forward-scattering)
    "C10 cos sign": ("double P = orc_hg((double)med->hg_g, dot3(Ln[l], f));",
                     "double P = orc_hg((double)med->hg_g, -dot3(Ln[l], f));", None, None),
    # C7 RIEMANN: A_n without the step length
    "C7 RIEMANN no h": ("else if (m->opacity_form == 1) A = alpha * T_prev * s;",
                        "else if (m->opacity_form == 1) A = alpha * T_prev * sigma_t;", None, None),
    "C6 >= instead of >": ("if ((float)sigma_s > m->depth_tau) { n_hit = (uint32_t)n; Dout = t; }",
                           "if ((float)sigma_s >= m->depth_tau) { n_hit = (uint32_t)n; Dout = t; }", None, None),
}


def main():
    keep = "--keep" in sys.argv
    tmp = tempfile.mkdtemp(prefix="nsl_mut_")
    files = subprocess.run(["git", "ls-files"], cwd=ROOT, capture_output=True, text=True).stdout.split()
    for f in files:
        d = os.path.join(tmp, os.path.dirname(f))
        os.makedirs(d, exist_ok=True)
        shutil.copy2(os.path.join(ROOT, f), os.path.join(tmp, f))
    src = os.path.join(tmp, "oracle", "nsl_oracle.c")
    orig = open(src).read()
    ok = True
    for name, (a, b, c, d) in MUTANTS.items():
        s = orig
        assert a in s, name
        s = s.replace(a, b, 1)
        if c:
            assert c in s, name
            s = s.replace(c, d, 1)
        open(src, "w").write(s)
        for so in ("libnsl_oracle.so",):
            p = os.path.join(tmp, "oracle", so)
            if os.path.exists(p):
                os.remove(p)
        r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-x", "-p",
                            "no:cacheprovider"], cwd=tmp, capture_output=True, text=True)
        killed = r.returncode != 0
        failed = [l.split("::")[-1].split(" ")[0] for l in r.stdout.splitlines() if l.startswith("FAILED")]
        print(f"{name:28s} {'killed' if killed else 'SURVIVED'} {failed}", flush=True)
        ok &= killed
    open(src, "w").write(orig)
    if not keep:
        shutil.rmtree(tmp)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
