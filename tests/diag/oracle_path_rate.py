"""The CPU oracle's own k-point throughput on a whole band path (test infrastructure: imports oracle/ and
synth/ only): min(nk, cores) worker processes, OMP_NUM_THREADS=1 each, draw k-points from one queue and
solve them completely with O.eigs_iterative (SciPy LOBPCG on the oracle operator, the oracle's K_P^{-1},
guard 5) to the bench tolerance.  k-points/s = nk / wall.  No model, no extrapolation.

usage: OMP_NUM_THREADS=1 python tests/diag/oracle_path_rate.py C2 [--k 0,5,...] [--tol 1e-5] [--out f.json]
"""
import argparse
import json
import os
import platform
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def solve(args):
    wname, ki, tol = args
    import synth
    from oracle import pc_oracle as O
    W = synth.WORKLOADS[wname]
    t0 = time.time()
    op = O.PenalizedOperator(W.n, W.kpoints()[ki], W.A(), W.eps1(), W.masks(), "crossdof")
    info = {}
    ev, res = O.eigs_iterative(op, W.nev, tol=tol, seed=1000 + ki, maxiter=1000, guard=5, info=info)
    return {"kidx": ki, "seconds": time.time() - t0, "iterations": info.get("iterations"),
            "max_res": float(res.max()), "omega2": [float(v) for v in ev]}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--k", default="")
    ap.add_argument("--tol", type=float, default=1e-5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import synth
    W = synth.WORKLOADS[a.workload]
    ks = [int(s) for s in a.k.split(",") if s.strip()] or list(range(len(W.kpoints())))
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    nw = max(1, min(len(ks), cores))
    t0 = time.time()
    with ProcessPoolExecutor(max_workers=nw) as ex:
        rows = list(ex.map(solve, [(a.workload, k, a.tol) for k in ks]))
    wall = time.time() - t0
    out = {"workload": a.workload, "n": W.n, "nev": W.nev, "tol": a.tol, "k_indices": ks, "workers": nw,
           "host_cores": cores, "cpu": cpu_model(), "threads_per_worker": os.environ.get("OMP_NUM_THREADS"),
           "wall_s": wall, "kpoints_per_s": len(ks) / wall,
           "mean_iterations": sum(r["iterations"] for r in rows) / len(rows), "rows": rows}
    print(json.dumps({k: v for k, v in out.items() if k != "rows"}), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
