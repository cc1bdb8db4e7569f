"""Parity helpers: CUDA path (via the C ABI) vs the CPU oracle, per DESIGN.md §3.

Value channels: |gpu - oracle| <= max(1e-4 |oracle|, 1e-5) per channel.
Depth D and the six debug counters: bit-exact.  Tie pixels (oracle decision
margin < 1e-5 at the depth threshold or at T_min) may differ in n_hit/n_term;
they are counted and re-verified by re-running the oracle with the GPU's
decisions forced, which must then meet the value bar and match D bitwise.
"""
import numpy as np

import oracle

REL, ABS, TIE = 1e-4, 1e-5, 1e-5


def value_ok(g, o):
    return np.abs(g - o) <= np.maximum(REL * np.abs(o), ABS)


def compare_frame(w, f, g_rgbt, g_depth, g_dbg, pixels=None, vals=None, check_debug=True, max_ties_frac=1e-4,
                  dec=None):
    """g_*: numpy arrays for the whole frame ([H,W,4], [H,W], [H,W,6] or None).
    dec: [H,W,2] (n_hit, n_term) of a DEBUG run of the same frame, for launches without
    counters (the timed FAST path): its primary march is the same arithmetic, so these are the
    FAST launch's own decisions (callers check T and D bitwise against the DEBUG run first).
    Tie pixels whose decisions differ from the oracle's are re-verified by
    re-running the oracle with the GPU's n_hit/n_term forced; none is left unverified.
    Returns a small report dict; raises AssertionError on any parity failure."""
    H, W = w.height, w.width
    if pixels is None:
        pixels = np.arange(H * W, dtype=np.int64)
    pixels = np.asarray(pixels, np.int64)
    if vals is None:
        vals = w.volume(w.frame_vol[f])
    cam, lights = w.cameras[f], w.lights[f]
    ref = oracle.guiding_map(w.grid, vals, cam, lights, w.light_mode, w.medium, w.march,
                             frame_id=w.frame_ids[f], pixels=pixels)
    g = g_rgbt.reshape(-1, 4)[pixels].astype(np.float64)
    gd = g_depth.reshape(-1)[pixels]
    tie = (ref["margin"] < TIE).any(axis=1)
    gdbg = None if g_dbg is None else g_dbg.reshape(-1, 6)[pixels].astype(np.uint32)
    if gdbg is not None:
        gdec = gdbg[:, 2:4]
    elif dec is not None:
        gdec = np.asarray(dec).reshape(-1, 2)[pixels].astype(np.uint32)
    else:
        gdec = None
    dec_mismatch = gd != ref["depth"]
    if gdec is not None:
        dec_mismatch |= (gdec[:, 0] != ref["debug"][:, 2]) | (gdec[:, 1] != ref["debug"][:, 3])
    bad_dec = dec_mismatch & ~tie
    assert not bad_dec.any(), (
        f"{int(bad_dec.sum())} non-tie pixels differ in depth/n_hit/n_term, e.g. pixel "
        f"{pixels[bad_dec][0]}: gpu D={gd[bad_dec][0]!r} oracle D={ref['depth'][bad_dec][0]!r}")
    if gdec is None:
        # no decisions to force the oracle with: every pixel, ties included, must meet the
        # value bar and match D bitwise as it stands (nothing is excluded)
        dec_mismatch = np.zeros(len(pixels), bool)
    ok = ~dec_mismatch
    vo = value_ok(g[ok], ref["rgbt"][ok])
    if not vo.all():
        i = np.argwhere(~vo)[0]
        pi = pixels[ok][i[0]]
        raise AssertionError(f"value parity: pixel {pi} ch {i[1]} gpu {g[ok][i[0], i[1]]!r} "
                             f"oracle {ref['rgbt'][ok][i[0], i[1]]!r} ({int((~vo).sum())} bad entries, "
                             f"tie={bool(tie[ok][i[0]])})")
    assert np.array_equal(gd[ok], ref["depth"][ok])
    if gdbg is not None and check_debug:
        same = gdbg[ok] == ref["debug"][ok]
        if not same.all():
            i = np.argwhere(~same)[0]
            raise AssertionError(f"debug counter {i[1]} differs at pixel {pixels[ok][i[0]]}: "
                                 f"gpu {gdbg[ok][i[0]]} oracle {ref['debug'][ok][i[0]]}")
    n_rever = int(dec_mismatch.sum())
    if n_rever:
        assert n_rever <= max(2, max_ties_frac * len(pixels)), f"too many tie pixels: {n_rever}"
        sub = pixels[dec_mismatch]
        fh = gdec[dec_mismatch, 0].astype(np.int32)
        ft = gdec[dec_mismatch, 1].astype(np.int32)
        r2 = oracle.guiding_map(w.grid, vals, cam, lights, w.light_mode, w.medium, w.march,
                                frame_id=w.frame_ids[f], pixels=sub, forced_hit=fh, forced_term=ft)
        assert value_ok(g[dec_mismatch], r2["rgbt"]).all(), "tie pixel failed forced re-verification"
        assert np.array_equal(gd[dec_mismatch], r2["depth"])
    err = np.abs(g - ref["rgbt"])
    return {"pixels": int(len(pixels)), "ties": int(tie.sum()), "reverified": n_rever,
            "unverified_ties": 0,
            "max_abs_err": float(err.max()) if len(err) else 0.0,
            "samples": int(((ref["debug"][:, 3] - ref["debug"][:, 0] + 1) * (ref["debug"][:, 0] > 0)).sum()
                           + ref["debug"][:, 5].sum())}


def fast_decisions(fast, debug, pixels=None):
    """(n_hit, n_term) per pixel of a FAST launch, from a DEBUG launch of the same frames.
    fast, debug: (rgbt [F,H,W,4], depth [F,H,W], dbg) numpy tuples.  Asserts first that the two
    launches agree bitwise on T and D (the primary march -- C5-C7, C11 -- is the same arithmetic
    in every kernel variant; only the light transmittances may differ, C9), which makes the
    DEBUG decisions the FAST launch's own."""
    fr, fd = np.asarray(fast[0]), np.asarray(fast[1])
    dr, dd, dbg = np.asarray(debug[0]), np.asarray(debug[1]), np.asarray(debug[2])
    F = fr.shape[0]
    for i in range(F):
        a, b = fr[i].reshape(-1, 4)[:, 3], dr[i].reshape(-1, 4)[:, 3]
        x, y = fd[i].reshape(-1), dd[i].reshape(-1)
        if pixels is not None:
            a, b, x, y = a[pixels], b[pixels], x[pixels], y[pixels]
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), f"frame {i}: FAST and DEBUG T differ"
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), f"frame {i}: FAST and DEBUG D differ"
    return dbg[..., 2:4]
