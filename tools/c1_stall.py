"""Vacuum n = 8 at k = (pi,pi,pi) from a Gaussian start (the degenerate-cluster case of the C1 test):
iterations and final residuals for several block shapes; max wanted residual every 25 iterations."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2511_17107_b200 import api  # noqa: E402

PI = math.pi
ctx = api.pc_create(np.eye(3), 8, np.eye(3), np.zeros((4, 8, 8, 8), np.uint8))
api.pc_set_option(ctx, "start", 0)
cases = [(6, 0, 1e-12), (10, 0, 1e-12), (10, -1, 1e-12), (6, -1, 1e-12), (8, 0, 1e-12)]
if len(sys.argv) > 1:
    cases = [(6, 0, float(d)) for d in sys.argv[1:]] + [(8, 0, float(d)) for d in sys.argv[1:]]
for g, wg, dt in cases:
    api.pc_set_option(ctx, "guard", g)
    api.pc_set_option(ctx, "w_guard", wg)
    api.pc_set_option(ctx, "drop_tol", dt)
    r = api.pc_bands(ctx, [[PI, PI, PI]], nev=6, tol=1e-7, maxit=500)
    h = api.pc_history(ctx)
    print(json.dumps({"guard": g, "w_guard": wg, "drop_tol": dt, "iters": int(r["iters"][0]), "status": int(r["status"][0]),
                      "res": r["resid"][0].tolist(),
                      "maxres_every_25": [float(h[i, :6].max()) for i in range(0, len(h), 25)]}), flush=True)
