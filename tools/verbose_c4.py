"""Per-iteration Res_j history of one C4 solve (bench workload, default options): active-column counts
per iteration and the iteration at which each wanted band converged (LOBPCG tail analysis)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api  # noqa: E402

W = synth.WORKLOADS["C4"]
ki = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = api.pc_create(W.A(), W.n, W.eps1(), W.masks())
api.pc_set_option(ctx, "kindex_offset", ki)
r = api.pc_bands(ctx, W.kpoints()[ki:ki + 1], nev=W.nev, tol=1e-5)
h = api.pc_history(ctx)
act = (h[:, :W.nev] > 1e-5).sum(axis=1)
conv_at = [int(np.argmax(h[:, j] <= 1e-5)) for j in range(W.nev)]
print(json.dumps({"kidx": ki, "iters": int(r["iters"][0]), "active_per_iter": act.tolist(),
                  "band_converged_at": conv_at, "iters_with_active_le_2": int((act <= 2).sum()),
                  "iters_with_active_le_5": int((act <= 5).sum())}))
