"""k-points/s of lock-step batches (option kbatch) against one-at-a-time solves and against
concurrent contexts, on the small configurations (C2 n = 32, C3 n = 64)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api, bands  # noqa: E402

wname = sys.argv[1] if len(sys.argv) > 1 else "C2"
nk = int(sys.argv[2]) if len(sys.argv) > 2 else 16
W = synth.WORKLOADS[wname]
kp = W.kpoints()
idx = list(range(1, 1 + nk))
out = {"workload": wname, "n": W.n, "nk": nk}
for kb in (1, 4, 8, 12):
    ctx = api.pc_create(W.A(), W.n, W.eps1(), W.masks())
    api.pc_set_option(ctx, "kbatch", kb)
    api.pc_bands(ctx, kp[1:1 + kb], nev=W.nev, tol=1e-5)  # warm-up
    api.pc_set_option(ctx, "kindex_offset", 1)
    torch.cuda.synchronize()
    t = time.time()
    r = api.pc_bands(ctx, kp[idx], nev=W.nev, tol=1e-5)
    torch.cuda.synchronize()
    out[f"kbatch{kb}"] = {"kpts_per_s": nk / (time.time() - t), "iters_mean": float(r["iters"].mean())}
    ctx.close()
for ncx in (2, 4):
    ctxs = [api.pc_create(W.A(), W.n, W.eps1(), W.masks()) for _ in range(ncx)]
    bands.solve_concurrent(ctxs, kp, [1] * ncx, W.nev, 1e-5, 500, 0)
    torch.cuda.synchronize()
    t = time.time()
    om, rs, it, stt = bands.solve_concurrent(ctxs, kp, idx, W.nev, 1e-5, 500, 0)
    torch.cuda.synchronize()
    out[f"contexts{ncx}"] = {"kpts_per_s": nk / (time.time() - t), "iters_mean": float(it.mean())}
    for c in ctxs:
        c.close()
print(json.dumps(out))
