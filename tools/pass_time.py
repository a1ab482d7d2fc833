"""CUDA-event time of single FFT passes at the bench workload (C4, n=128, 15 columns): the plain
y/z/x passes and the two symbol-fused z passes of pc_apply (tuning aid)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api  # noqa: E402

W = synth.WORKLOADS["C4"]
ncol = int(sys.argv[1]) if len(sys.argv) > 1 else 15
A = W.A()
ctx = api.pc_create(A, W.n, W.eps1(), synth.make_masks(W.geometry, A, W.n))
X = torch.randn(ncol, 3 * W.n ** 3, dtype=torch.complex128, device="cuda")
Y = torch.empty_like(X)
k = W.kpoints()[5]
pts = W.n ** 3 * ncol
out = {}
for name, kind, axis, d, xh, byt in [("z_plain", 0, 2, 1, None, 96), ("y_plain", 0, 1, 1, None, 96),
                                     ("x_plain", 0, 0, 1, None, 96), ("z_kah", 1, 2, 1, None, 96),
                                     ("z_ka", 2, 2, -1, X, 144)]:
    for _ in range(2):
        api.pc_debug_pass(ctx, k, kind, axis, d, X, Y, xh)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record()
        api.pc_debug_pass(ctx, k, kind, axis, d, X, Y, xh)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    out[name] = {"ms": round(ms, 4), "gbs": round(byt * pts / ms / 1e6, 1)}
print(json.dumps(out))
