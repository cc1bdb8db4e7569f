"""CPU simulation of L1 line traffic of the light-march gathers for candidate
volume layouts (layout design study).  Reproduces the kernel's
sample positions for C2 frame 0 (frame constants and jitter from the oracle's
helpers, fp32 numpy), groups lanes exactly as a warp does (8x4 pixel tile,
lock-step primary step index), and counts distinct 128-B lines touched by each
warp-wide gather instruction under each layout."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import nsl_inputs as I  # noqa: E402
import oracle  # noqa: E402

w = I.make_workload("C2", frames=[int(sys.argv[1]) if len(sys.argv) > 1 else 0])
vals = w.volume(0)
n = w.grid.nx
fc = oracle.frame_constants(w.grid, w.cameras[0], w.lights[0], w.light_mode, w.medium, w.march)
W = H = 512
h = np.float32(w.march.step)
py, px = np.mgrid[0:H, 0:W].astype(np.float32)
B, Ex, Ey, Dg = fc["B"], fc["Ex"], fc["Ey"], fc["Dg"]
O = [(py * Ey[a] + (px * Ex[a] + B[a])).astype(np.float32) for a in range(3)]   # (fma vs mul+add: close enough)
pix = (np.arange(H)[:, None] * W + np.arange(W)[None, :]).astype(np.int64)
delta = np.array([oracle.jitter_delta(w.march, 0, int(p)) for p in pix.reshape(-1)], np.float32).reshape(H, W)

pad = np.zeros((n + 2, n + 2, n + 2), np.float32)
pad[1:-1, 1:-1, 1:-1] = vals
cellnz = (pad[:-1, :-1, :-1] + pad[1:, :-1, :-1] + pad[:-1, 1:, :-1] + pad[1:, 1:, :-1] +
          pad[:-1, :-1, 1:] + pad[1:, :-1, 1:] + pad[:-1, 1:, 1:] + pad[1:, 1:, 1:]) > 0   # [z][y][x], cells 0..n

def rho_occ(x, y, z):
    ok = (x > 0) & (x < n + 1) & (y > 0) & (y < n + 1) & (z > 0) & (z < n + 1)
    ix, iy, iz = np.floor(x).astype(int), np.floor(y).astype(int), np.floor(z).astype(int)
    out = np.zeros(x.shape, bool)
    out[ok] = cellnz[iz[ok], iy[ok], ix[ok]]
    return out, ix, iy, iz

LAYOUTS = {
    # name: function (ix, iy, iz) -> list of line ids per gather instruction
    "quad_f32 x-linear (2 x LDG.128)": lambda i, j, k: [((k * (n + 1) + j) * (n + 1) + i) * 16 // 128,
                                                        (((k + 1) * (n + 1) + j) * (n + 1) + i) * 16 // 128],
    "quad_f32 2x2x2 bricks (2 x LDG.128)": lambda i, j, k: [brick(i, j, k, 2, 2, 2, 16), brick(i, j, k + 1, 2, 2, 2, 16)],
    "quad_f32 4x2x1 bricks (2 x LDG.128)": lambda i, j, k: [brick(i, j, k, 4, 2, 1, 16), brick(i, j, k + 1, 4, 2, 1, 16)],
    "corner_f16 x-linear (1 x LDG.128)": lambda i, j, k: [((k * (n + 1) + j) * (n + 1) + i) * 16 // 128],
    "corner_f16 2x2x2 bricks (1 x LDG.128)": lambda i, j, k: [brick(i, j, k, 2, 2, 2, 16)],
    "linear_f32 (8 x LDG.32)": lambda i, j, k: [((k + dk) * (n + 2) + (j + dj)) * (n + 2) + i + di
                                                for dk in (0, 1) for dj in (0, 1) for di in (0, 1)],
}
LAYOUTS["linear_f32 (8 x LDG.32)"] = lambda i, j, k: [(((k + dk) * (n + 2) + (j + dj)) * (n + 2) + i + di) * 4 // 128
                                                      for dk in (0, 1) for dj in (0, 1) for di in (0, 1)]


def brick(i, j, k, bx, by, bz, esz):
    nbx, nby = (n + 2 + bx - 1) // bx, (n + 2 + by - 1) // by
    b = ((k // bz) * nby + j // by) * nbx + i // bx
    inner = ((k % bz) * by + j % by) * bx + i % bx
    return (b * (bx * by * bz) + inner) * esz // 128


stats = {k: [0, 0] for k in LAYOUTS}   # lines, warp-instructions
hl = h
Lg = fc["Lg"]
for ty in range(0, H, 4):
    for tx in range(0, W, 8):
        sl = (slice(ty, ty + 4), slice(tx, tx + 8))
        ox, oy, oz = O[0][sl].reshape(-1), O[1][sl].reshape(-1), O[2][sl].reshape(-1)
        d = delta[sl].reshape(-1)
        for nstep in range(1, 40):
            t = (np.float32(nstep) * h + d).astype(np.float32)
            x = (t * Dg[0] + ox).astype(np.float32)
            y = (t * Dg[1] + oy).astype(np.float32)
            z = (t * Dg[2] + oz).astype(np.float32)
            occ, _, _, _ = rho_occ(x, y, z)
            if not occ.any():
                continue
            for l in (1, 2):
                for j in range(1, 30):
                    s = np.float32(j) * hl
                    X = (s * Lg[l][0] + x).astype(np.float32)
                    Y = (s * Lg[l][1] + y).astype(np.float32)
                    Z = (s * Lg[l][2] + z).astype(np.float32)
                    o2, ix, iy, iz = rho_occ(X, Y, Z)
                    act = occ & o2
                    if not act.any():
                        if not (occ & (X > 0) & (X < n + 1) & (Y > 0) & (Y < n + 1)).any():
                            break
                        continue
                    for name, f in LAYOUTS.items():
                        lines = f(ix[act], iy[act], iz[act])
                        for arr in lines:
                            stats[name][0] += len(np.unique(arr))
                            stats[name][1] += 1
for name, (lines, instr) in stats.items():
    print(f"{name:42s} warp-gather instructions {instr:9d}  lines/instr {lines / max(instr, 1):6.2f}  "
          f"lines per warp-sample {lines / max(stats['corner_f16 x-linear (1 x LDG.128)'][1], 1):6.2f}")
