"""one multi-k launch sequence (pc_apply_multi / pc_precond_multi: k as an extra column
dimension) against one pc_apply / pc_precond per k-point, on the small configurations (C2 n = 32,
C3 n = 64) where one k-point's block under-fills the GPU.

usage: python tools/multik_time.py [C2] [--nk 8] [--cols 10]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="C2")
ap.add_argument("--nk", type=int, default=8)
ap.add_argument("--cols", type=int, default=10)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
W = synth.WORKLOADS[a.workload]
ctx = api.pc_create(W.A(), W.n, W.eps1(), W.masks())
kp = W.kpoints()[1:1 + a.nk]
kcol = [j // a.cols for j in range(a.nk * a.cols)]
X = torch.randn(len(kcol), 3 * W.n ** 3, dtype=torch.complex128, device="cuda")
Y = torch.empty_like(X)
Y1 = torch.empty_like(X)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


def per_k_apply():
    for i in range(a.nk):
        api.pc_apply(ctx, kp[i], X[i * a.cols:(i + 1) * a.cols], Y1[i * a.cols:(i + 1) * a.cols])


def per_k_precond():
    for i in range(a.nk):
        api.pc_precond(ctx, kp[i], X[i * a.cols:(i + 1) * a.cols], Y1[i * a.cols:(i + 1) * a.cols])


out = {"workload": a.workload, "n": W.n, "nk": a.nk, "cols_per_k": a.cols}
out["apply_multi_ms"] = timed(lambda: api.pc_apply_multi(ctx, kp, kcol, X, Y))
out["apply_per_k_ms"] = timed(per_k_apply)
out["precond_multi_ms"] = timed(lambda: api.pc_precond_multi(ctx, kp, kcol, X, Y))
out["precond_per_k_ms"] = timed(per_k_precond)
api.pc_apply_multi(ctx, kp, kcol, X, Y)
per_k_apply()
out["max_rel_diff"] = float(torch.max(torch.linalg.vector_norm(Y - Y1, dim=1) / torch.linalg.vector_norm(Y1, dim=1)))
pts = W.n ** 3 * len(kcol)
out["apply_multi_alg_gbs"] = 336 * pts / out["apply_multi_ms"] / 1e6
out["apply_per_k_alg_gbs"] = 336 * pts / out["apply_per_k_ms"] / 1e6
print(json.dumps(out))
