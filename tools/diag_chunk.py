import sys, math, numpy as np, torch
sys.path.insert(0, '.')
import synth
from paper_2511_17107_b200 import api
W = synth.WORKLOADS["C4"]
n = W.n; A = W.A()
masks = W.masks()
ctx = api.pc_create(A, n, W.eps1(), masks)
k = [math.pi, math.pi, math.pi]
for ncol in (10, 15):
    X = torch.randn(ncol, 3 * n**3, dtype=torch.complex128, device="cuda")
    Y0 = torch.empty_like(X); Y = torch.empty_like(X)
    api.pc_set_option(ctx, "chunk_mb", 0); api.pc_apply(ctx, k, X, Y0)
    for cmb in (0, 12, 24, 48, 96, 200):
        api.pc_set_option(ctx, "chunk_mb", cmb)
        for _ in range(3): api.pc_apply(ctx, k, X, Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5): api.pc_apply(ctx, k, X, Y)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        err = ((Y - Y0).norm() / Y0.norm()).item()
        print(f"ncol {ncol} chunk_mb {cmb}: {ms:.3f} ms  alg {336*n**3*ncol/ms/1e6:.0f} GB/s  err {err:.1e}", flush=True)
