"""Rayleigh-Ritz phase cycles and Jacobi sweeps per LOBPCG iteration (needs a -DPC_RR_TIMING build of
libpcband: PCBAND_LIB=var/<v>/libpcband.so).  Runs one k-point with option verbose = 1 and parses the
per-iteration '[pcband] ... sweeps S ... rr-cycles a b c d e' lines (scaling, Cholesky, H formation,
Jacobi, back substitution) from stderr of a child process.

usage: python tools/rr_phases.py [C4] [kidx] [maxit]"""
import json
import os
import re
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import synth
    from paper_2511_17107_b200 import api
    W = synth.WORKLOADS[sys.argv[2]]
    ki, maxit = int(sys.argv[3]), int(sys.argv[4])
    ctx = api.pc_create(W.A(), W.n, W.eps1(), W.masks())
    api.pc_set_option(ctx, "verbose", 1)
    api.pc_set_option(ctx, "kindex_offset", ki)
    api.pc_bands(ctx, W.kpoints()[ki:ki + 1], nev=W.nev, tol=1e-5, maxit=maxit)
    sys.exit(0)

wl = sys.argv[1] if len(sys.argv) > 1 else "C4"
ki = sys.argv[2] if len(sys.argv) > 2 else "5"
maxit = sys.argv[3] if len(sys.argv) > 3 else "1000"
p = subprocess.run([sys.executable, __file__, "--child", wl, ki, maxit], capture_output=True, text=True)
rows = []
for line in p.stderr.splitlines():
    m = re.search(r"sweeps (\d+) .*rr-cycles (\d+) (\d+) (\d+) (\d+) (\d+)", line)
    if m:
        rows.append([int(x) for x in m.groups()])
if not rows:
    print(p.stderr[-2000:])
    sys.exit(1)
n = len(rows)
mean = [sum(r[i] for r in rows) / n for i in range(6)]
print(json.dumps({"workload": wl, "kidx": int(ki), "iterations": n, "mean_sweeps": mean[0],
                  "mean_cycles": {"scaling": mean[1], "cholesky": mean[2], "h_formation": mean[3],
                                  "jacobi": mean[4], "back_substitution": mean[5]},
                  "sweeps_hist": {s: sum(1 for r in rows if r[0] == s) for s in sorted(set(r[0] for r in rows))}}))
