"""Per-pass CUDA-event times of one 15-column pc_apply at the bench workload (C4, n=128).

usage: python tools/apply_time.py [C4] [ncols] [key=value ...]   (eps=sdd: the general eps_1 with all three
       off-diagonal couplings, which runs the 7-pass path with the standalone stencil)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api  # noqa: E402

W = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ncol = int(sys.argv[2]) if len(sys.argv) > 2 else 15
A = W.A()
masks = synth.make_masks(W.geometry, A, W.n)
opts = dict(kv.split("=") for kv in sys.argv[3:])  # extra key=value options
eps1 = synth.eps_sdd() if opts.pop("eps", "") == "sdd" else W.eps1()
ctx = api.pc_create(A, W.n, eps1, masks)
for key, v in opts.items():
    api.pc_set_option(ctx, key, float(v))
X = torch.randn(ncol, 3 * W.n ** 3, dtype=torch.complex128, device="cuda")
Y = torch.empty_like(X)
k = W.kpoints()[5]
for _ in range(3):
    api.pc_apply(ctx, k, X, Y)
api.pc_set_option(ctx, "profile", 1)
api.pc_stats(ctx, reset=True)
reps = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    api.pc_apply(ctx, k, X, Y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
st = api.pc_stats(ctx)
pts = W.n ** 3 * ncol
design = sum(v["bytes"] for v in st.values() if isinstance(v, dict)) / reps / pts  # B per point per column
out = {"ms": ms, "alg_gbs": 336 * pts / ms / 1e6, "design_bytes_per_point": design, "design_gbs": design * pts / ms / 1e6,
       "classes": {k_: round(v["ms"] / reps, 4) for k_, v in st.items() if isinstance(v, dict) and v["count"]}}
print(json.dumps(out))
