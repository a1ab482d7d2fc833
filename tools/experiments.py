"""Round-1 experiments on the CUDA path, synthetic geometries.

f1  M_Trivial vs M_CrossDoF (Table 1 analogue): Delta omega_max / mean over the
    full band path (omega = sqrt(omega^2)), mean/std LOBPCG iterations (Table 2
    analogue), gap ratio for SC-CURV, FCC diamond, BCC-SG, BCC-DG.
f3  ill-conditioned eps_1 = U diag(1e-1, 1e-3, 1e-5) U^H on SC-CURV at k = (1/7, 3/5, 4/13) pi
    (P:1284-1299): iterations and the asymptotic damping factor theta from a linear regression of
    log residuals, Trivial vs CrossDoF (this eps_1 couples all three components, so the
    general 7-pass apply path with the full CrossDoF stencil runs).

usage: python tools/experiments.py [--n 64] [--segments 8] [--streams 4] > profiles/r01_experiments.json
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_17107_b200 import api, bands  # noqa: E402

PI = math.pi


def solve_path(A, n, eps1, masks, mode, kp, nev, tol, streams, maxit=1000):
    ctxs = [api.pc_create(A, n, eps1, masks, eps_mode=mode) for _ in range(streams)]
    t = time.time()
    om, rs, it, st = bands.solve_concurrent(ctxs, kp, list(range(len(kp))), nev, tol, maxit, 0)
    el = time.time() - t
    for c in ctxs:
        c.close()
    return om, it, st, el


def gap_ratio(om):
    w = np.sqrt(np.maximum(om, 0))
    best = (0.0, None)
    for j in range(w.shape[1] - 1):
        low, up = w[:, j].max(), w[:, j + 1].min()
        if up > low:
            r = (up - low) / ((up + low) / 2)
            if r > best[0]:
                best = (r, j + 1)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--segments", type=int, default=8)
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--tol", type=float, default=1e-5)
    a = ap.parse_args()
    nev = 10
    out = {"n": a.n, "nev": nev, "tol": a.tol, "segments": a.segments, "f1": {}, "f3": {}}
    cases = [("SC-CURV", "sc", "sc_curv", 13.0), ("FCC", "fcc", "fcc_diamond", 13.0),
             ("BCC-SG", "bcc", "bcc_sg", 16.0), ("BCC-DG", "bcc", "bcc_dg", 16.0)]
    for name, lat, geo, el in cases:
        A = synth.lattice(lat)
        masks = synth.make_masks(geo, A, a.n)
        kp = synth.kpath(lat, a.segments)
        row = {"fill": float(masks[3].mean()), "nk": len(kp)}
        res = {}
        for tag, eps1, mode in (("iso", synth.eps_isotropic(el), "crossdof"),
                                ("trivial", synth.eps_pseudochiral(el, 0.875), "trivial"),
                                ("crossdof", synth.eps_pseudochiral(el, 0.875), "crossdof")):
            om, it, st, t = solve_path(A, a.n, eps1, masks, mode, kp, nev, a.tol, a.streams)
            res[tag] = om
            g = gap_ratio(om)
            row[tag] = {"iters_mean": float(it.mean()), "iters_std": float(it.std()),
                        "unconverged": int((st != 0).sum()), "seconds": t,
                        "gap_ratio": g[0], "gap_above_band": g[1]}
        w1, w2 = np.sqrt(res["trivial"]), np.sqrt(res["crossdof"])
        d = np.abs(w1 - w2) / np.abs(w2)
        row["domega_max"] = float(d.max())
        row["domega_mean"] = float(d.mean())
        out["f1"][name] = row
        print(name, json.dumps(row), file=sys.stderr, flush=True)

    # f3: ill-conditioned eps_1 on SC-CURV at k = (1/7, 3/5, 4/13) pi
    A = synth.lattice("sc")
    masks = synth.make_masks("sc_curv", A, a.n)
    eps1 = synth.eps_extreme(7)
    k = np.array([1 / 7, 3 / 5, 4 / 13]) * PI
    for mode in ("trivial", "crossdof"):
        ctx = api.pc_create(A, a.n, eps1, masks, eps_mode=mode)
        t = time.time()
        r = api.pc_bands(ctx, [k], nev=nev, tol=a.tol, maxit=2000)
        el = time.time() - t
        h = api.pc_history(ctx)[:, :nev].max(axis=1)
        m = len(h)
        tail = np.arange(m // 2, m)
        slope = np.polyfit(tail, np.log(h[tail]), 1)[0] if len(tail) > 2 else float("nan")
        out["f3"][mode] = {"iters": int(r["iters"][0]), "status": int(r["status"][0]), "seconds": el,
                           "theta": float(math.exp(slope)), "omega2": r["omega2"][0].tolist(),
                           "hpd_flags": api.pc_info(ctx)["hpd_flags"],
                           "residual_history_max": h[:: max(1, m // 40)].tolist()}
        ctx.close()
        print(mode, out["f3"][mode]["iters"], out["f3"][mode]["theta"], file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
