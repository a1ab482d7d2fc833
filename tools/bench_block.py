"""Isolated timing of the LOBPCG block kernels (pc_bench_block) at the bench shape (n=128, b=15,
na = nP = 10): fused update (which 0; 3 = TMA tensor-copy variant), Gram S^H[W P AW AP] (1), Gram S^H[W AW] (2), with HBM GB/s of
the algorithmic traffic.  PCBAND_LIB selects a variant build.

usage: python tools/bench_block.py [--n 128] [--b 15] [--na 10] [--np 10] [--reps 20] [--which 0 1]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--b", type=int, default=15)
ap.add_argument("--na", type=int, default=10)
ap.add_argument("--np", type=int, default=10)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--which", type=int, nargs="+", default=[0, 1])
ap.add_argument("--opt", nargs=2, action="append", default=[])
a = ap.parse_args()
A = synth.lattice("fcc")
ctx = api.pc_create(A, a.n, synth.eps_pseudochiral(), synth.make_masks("fcc_diamond", A, a.n))
for k, v in a.opt:
    api.pc_set_option(ctx, k, float(v))
rows = 3 * a.n ** 3
p = a.b + a.na + a.np
out = {}
for w in a.which:
    ms = api.pc_bench_block(ctx, w, a.b, a.na, a.np, a.reps)
    if w in (0, 3):
        cols = 2 * p + 2 * a.b + 3 * a.na
    elif w in (1, 4):
        cols = p + 2 * (a.na + a.np)
    else:
        cols = p + a.na
    out[w] = {"ms": round(ms, 4), "gbs": round(16.0 * rows * cols / ms / 1e6, 1), "cols": cols}
    if w == 1:  # algorithmic Gram flops: p x 2c complex MACs per row, 8 flops each
        out[w]["alg_tflops"] = round(8.0 * rows * p * 2 * (a.na + a.np) / ms / 1e9, 2)
print(json.dumps(out))
