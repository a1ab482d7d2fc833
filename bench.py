#!/usr/bin/env python
"""Benchmark: k-points/s of the full 10-band pseudochiral band solve at n = 128 (BASELINE.json metric,
config 4 of BASELINE.json: FCC lattice, diamond inclusion, eps_1 pseudochiral, tol 1e-5 as in
PAPER.md:1064), plus the pc_apply HBM bandwidth.

    python bench.py [--gpus N --steps K --warmup W]                     # our arm (libpcband.so)
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N   # N > 1 (NCCL)
    python bench.py --impl reference                                    # the CPU oracle arm

A step = one Bloch vector solved to tolerance by pc_bands (symbols, K_A^H/FFT/M_eps/FFT/K_A applies,
K_P^{-1}, Gram, Rayleigh-Ritz, updates -- every row of SURVEY §8(a)).  Each rank solves K distinct
k-points of the 49-point path (weak scaling); value = all ranks' k-points / max-over-ranks time.
One JSON line is printed by rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "k-points/sec (10 bands, n=128, FP64) and pc_apply HBM GB/s vs 8 TB/s"
PAPER_ITERS_FCC_PC = 51.3   # mean LOBPCG iterations, pseudochiral FCC, CrossDoF, N=120


def load_json(path, default=None):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return default


def peaks():
    mp = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"), {}) or {}
    fp = load_json(os.path.join(ROOT, "profiles", "fp64_peaks.json"), {}) or {}
    hbm = mp.get("hbm_gbs")
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (measured)"
    if hbm is None:
        hbm, hbm_src = 6650.0, "B200_PROFILING.md fallback"
    fp64 = fp.get("dmma_m8n8k4_tflops")
    fp64_src = "profiles/fp64_peaks.json (DMMA m8n8k4 microbenchmark, measured on this pool)"
    if fp64 is None:
        bf = mp.get("bf16_tflops", 1590.0)
        fp64, fp64_src = bf * 40.0 / 2250.0, "bf16 measured peak x nominal fp64/bf16 ratio (40/2250)"
    return hbm, hbm_src, fp64, fp64_src


# ------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.gpu)], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.strip().split(", ") for r in self.f.read().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference): the oracle as it stands, in worker processes
# (one per host core used, OMP_NUM_THREADS=1 each), on bounded samples of the workload.
# ------------------------------------------------------------------------------------------
def oracle_sample(W, k, nsample_cols=1, masks=None):
    """Time the oracle on a bounded sample of one k-point solve of workload W: sparse assembly of
    Op(k), nsample_cols Fourier-space applies + K_P^{-1} solves, and one Rayleigh-Ritz Gram of the
    3b-column block (b = nev + 5, the oracle's guard).  Returns the component times."""
    from oracle import pc_oracle as O
    import synth
    t0 = time.perf_counter()
    if masks is None:
        masks = W.masks()
    op = O.PenalizedOperator(W.n, k, W.A(), W.eps1(), masks)
    t_asm = time.perf_counter() - t0
    x = synth.random_block(W.n, nsample_cols, seed=3)
    t0 = time.perf_counter()
    y = op.apply_fourier(x)
    t_apply = (time.perf_counter() - t0) / nsample_cols
    t0 = time.perf_counter()
    O.precond_fourier(W.n, k, op.A, op.gamma, y)
    t_prec = (time.perf_counter() - t0) / nsample_cols
    b = W.nev + 5
    # one Gram S^H [S AS] of the 3b-column basis on the full vectors (numpy/BLAS), timed on a slab
    rows = min(op.dim, 1 << 18)
    S = np.random.default_rng(0).standard_normal((rows, 3 * b)) + 0j
    t0 = time.perf_counter()
    S.conj().T @ np.concatenate([S, S], axis=1)
    t_gram = (time.perf_counter() - t0) * (op.dim / rows)
    return {"assembly_s": t_asm, "apply_s_per_col": t_apply, "precond_s_per_col": t_prec,
            "gram_s": t_gram, "block": b}


def oracle_kpoint_s(t, iters):
    """Model of one oracle k-point solve: assembly + iters x (b applies + b K_P^{-1} + 2 Grams)."""
    b = t["block"]
    per_it = b * (t["apply_s_per_col"] + t["precond_s_per_col"]) + 2.0 * t["gram_s"]
    return t["assembly_s"] + iters * per_it, per_it


def oracle_iters(W):
    """The ORACLE's own LOBPCG iteration count on this workload (tests/diag/oracle_iters.py, committed
    under profiles/): SciPy LOBPCG on the oracle operator, tol 1e-5, guard 5.  None if not measured."""
    d = load_json(os.path.join(ROOT, "profiles", f"oracle_iters_{W.name.lower()}.json"), None)
    if not d or not d.get("rows"):
        return None, None
    its = [r["iterations"] for r in d["rows"]]
    grid = f", measured on the n = {d['n']} grid of the same geometry (the count barely depends on n: the device " \
           f"needs 82 / 85 / 89 at n = 32 / 64 / 128)" if d.get("grid_override") else ""
    return float(np.mean(its)), (f"profiles/oracle_iters_{W.name.lower()}.json: tol {d['rows'][0]['tol']:g}, "
                                 f"k {[r['kidx'] for r in d['rows']]}, iterations {its}{grid}")


def oracle_worker(args):
    """--oracle-worker (a subprocess, OMP_NUM_THREADS=1): component sample of workload args.workload at
    path point args.kidx, and optionally one complete oracle solve of a C2 path point (args.c2k)."""
    import synth
    from oracle import pc_oracle as O
    W = synth.WORKLOADS[args.workload]
    out = {"kidx": args.kidx, "components": oracle_sample(W, W.kpoints()[args.kidx])}
    if args.c2k >= 0:
        W2 = synth.WORKLOADS["C2"]
        t0 = time.perf_counter()
        op = O.PenalizedOperator(W2.n, W2.kpoints()[args.c2k], W2.A(), W2.eps1(), W2.masks())
        info = {}
        ev, res = O.eigs_iterative(op, W2.nev, tol=args.tol, seed=1000 + args.c2k, maxiter=600, guard=5, info=info)
        out["c2"] = {"kidx": args.c2k, "seconds": time.perf_counter() - t0, "iterations": info.get("iterations"),
                     "max_res": float(res.max())}
    print(json.dumps(out), flush=True)


def oracle_parallel(args, kidx_list, c2_list=None):
    """Run len(kidx_list) oracle workers at once (one per core, OMP_NUM_THREADS=1 each); returns their
    JSON results and the wall time."""
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE"):
        env.pop(k, None)
    procs = []
    t0 = time.perf_counter()
    for i, ki in enumerate(kidx_list):
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--oracle-worker", "--workload", args.workload,
               "--kidx", str(ki), "--tol", str(args.tol), "--c2k", str(c2_list[i] if c2_list else -1)]
        procs.append(subprocess.Popen(cmd, env=env, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True))
    outs = []
    for pr in procs:
        o, _ = pr.communicate()
        lines = [ln for ln in o.splitlines() if ln.startswith("{")]
        if pr.returncode != 0 or not lines:
            raise RuntimeError(f"oracle worker failed (rc {pr.returncode})")
        outs.append(json.loads(lines[-1]))
    return outs, time.perf_counter() - t0


def host_cores():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_baseline(args, W, steps_kidx, with_c2):
    """Oracle k-points/s on the host cores: nw = min(cores, 8) worker processes each time a component
    sample of a different k-point; a k-point's time is extrapolated with the oracle's own iteration
    count; value = nw / mean k-point time (nw k-points solved side by side).  with_c2: each worker also
    solves one C2 path point completely (a real oracle solve, no model): C2 k-points/s = nw / wall."""
    nw = max(1, min(host_cores(), 8))
    its, its_src = oracle_iters(W)
    nk = len(W.kpoints())
    kl = [steps_kidx[i % len(steps_kidx)] for i in range(nw)]
    c2l = [(3 * i + 1) % 33 for i in range(nw)] if with_c2 else None
    outs, wall = oracle_parallel(args, kl, c2l)
    comps = [o["components"] for o in outs]
    if its is None:
        its, its_src = PAPER_ITERS_FCC_PC, "PAPER.md:1199 (oracle count not measured)"
    ks = [oracle_kpoint_s(c, its)[0] for c in comps]
    value = nw / float(np.mean(ks))
    res = {"value": value, "unit": "k-points/s", "cores": nw, "kind": "oracle", "cpu": cpu_model(),
           "sample": (f"{nw} oracle worker processes (OMP_NUM_THREADS=1), each: sparse assembly of Op(k) at "
                      f"n={W.n} + 1 Fourier-space apply + 1 K_P^-1 column + one 3b-column Gram (b = nev + 5) "
                      f"at its own {W.name} path point; k-point time = assembly + {its:.0f} iterations (the oracle's "
                      f"own SciPy LOBPCG count, {its_src}) x (b applies + b K_P^-1 + 2 Grams); "
                      f"value = {nw} / mean k-point time"),
           "components_mean": {k: float(np.mean([c[k] for c in comps])) for k in comps[0]},
           "kpoint_s_mean": float(np.mean(ks)), "wall_s": wall, "nk_path": nk}
    if with_c2:
        c2 = [o["c2"] for o in outs]
        res["c2_measured"] = {"value": nw / max(c["seconds"] for c in c2), "unit": "k-points/s",
                              "what": f"{nw} complete oracle solves of C2 path points (SC sphere, n = 32, 10 bands, "
                                      f"tol {args.tol:g}) side by side, k-points / wall (no model)",
                              "iterations": [c["iterations"] for c in c2],
                              "seconds": [round(c["seconds"], 2) for c in c2]}
    # complete oracle solves of whole paths, measured on the GPU box's host cores (tests/diag/oracle_path_rate.py)
    meas = {}
    for wn in ("c2", "c3"):
        d = load_json(os.path.join(ROOT, "profiles", f"r02_oracle_path_{wn}.json"), None)
        if d:
            meas[wn.upper()] = {"kpoints_per_s": d["kpoints_per_s"], "k_points": len(d["k_indices"]),
                                "workers": d["workers"], "cpu": d["cpu"], "wall_s": d["wall_s"],
                                "mean_iterations": d["mean_iterations"], "tol": d["tol"],
                                "source": f"profiles/r02_oracle_path_{wn}.json"}
    if meas:
        res["measured_paths"] = meas
    res["paper_timings"] = ("context only: PAPER.md:1260 pseudochiral FCC N=120, 10 bands at (pi,pi,pi): "
                            "GPU 34.15 s (RTX 4090 D, cupy; 0.029 k-points/s), CPU 1506.35 s (numpy, CPU "
                            "model not stated; 0.00066 k-points/s), 55 LOBPCG steps")
    return res


def run_reference(args):
    """--impl reference: the CPU oracle arm (rank 0 only; other ranks exit 0).  Each step = one round of
    oracle workers (one per host core used) timing a component sample of different C4 path points."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    W = synth.WORKLOADS[args.workload]
    nk = len(W.kpoints())
    times, vals, last = [], [], None
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = oracle_baseline(args, W, [(s * 8 + i) % nk for i in range(8)], with_c2=False)
        el = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(el)
            vals.append(r["value"])
            last = r
    value = float(np.mean(vals))
    cpu = dict(last)
    cpu["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "k-points/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * float(np.mean(times)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(W, args), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "k-points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


PRECOND_DESC = {"kp": "K_P^{-1}, the paper's FFT-diagonal preconditioner (PAPER.md:530-548)",
                "eps": "eps-weighted K_P^{-1}: K_A^+H diag(M_eps)^{-1} K_A^+ + Pi/(gamma|kappa|^2) "
                       "(beyond the paper, DESIGN.md R16)"}


def workload_config(W, args):
    eps_desc = {"pc13": "pseudochiral eps_lat=13 beta=0.875, PAPER.md:1083-1093",
                "iso13": "isotropic eps_lat=13, PAPER.md:1082", "vacuum": "vacuum"}.get(W.eps, W.eps)
    return {"workload": f"{W.name}: {W.lattice.upper()} lattice, {W.geometry} inclusion, eps1={W.eps} "
                        f"({eps_desc}), n={W.n}, {W.nev} bands, "
                        f"tol={args.tol:g}, k-path {len(W.kpoints())} points",
            "n": W.n, "nev": W.nev, "block": W.nev + (args.guard if args.guard is not None else 6), "tol": args.tol, "lattice": W.lattice,
            "geometry": W.geometry, "eps_mode": "crossdof",
            "precond": PRECOND_DESC[getattr(args, "precond", "kp")],
            "l2": "no flush: per-k working set ~15 GB >> 126 MB L2",
            "start": ("warm: each context solves a contiguous k stretch, k_i started from k_(i-1)'s Ritz block "
                      "(SURVEY f2, not the paper's protocol)") if getattr(args, "warm_start", False)
            else "cold: seeded plane-wave + Gaussian start block per k"}


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--tol", type=float, default=1e-5)
    ap.add_argument("--maxit", type=int, default=500)
    ap.add_argument("--apply-cols", type=int, default=15)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--guard", type=int, default=None, help="LOBPCG guard columns (block = nev + guard)")
    ap.add_argument("--streams", type=int, default=2, help="concurrent k-point solves per GPU (contexts)")
    ap.add_argument("--kbatch", type=int, default=1,
                    help="k-points solved in lock step per pc_bands call (option kbatch; helps at n <= 64)")
    ap.add_argument("--w-guard", type=int, default=None, help="guard columns that get search directions")
    ap.add_argument("--warm-start", action="store_true",
                    help="path continuation: contiguous k stretches per context, each k started from the "
                         "previous k's Ritz block (SURVEY f2; not the paper's cold start, reported separately)")
    ap.add_argument("--precond", default="kp", choices=["kp", "eps"],
                    help="kp: the paper's K_P^{-1} (P:530-548, default, the headline); eps: the eps-weighted "
                         "preconditioner (beyond the paper, DESIGN R16)")
    ap.add_argument("--no-alt", action="store_true",
                    help="skip the secondary timed run with the other preconditioner (key alt_precond)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo + ranks sharing GPUs (rank -> device rank %% count): a functional test of the "
                         "multi-rank path on a smaller box; numbers from it are not scaling results")
    ap.add_argument("--cpu-c2", action="store_true",
                    help="cpu_baseline also runs complete oracle solves of C2 path points (1-2 min more)")
    ap.add_argument("--oracle-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--kidx", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--c2k", type=int, default=-1, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.oracle_worker:
        return oracle_worker(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import synth
    from paper_2511_17107_b200 import api, bands

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")  # collective buffers
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    W = synth.WORKLOADS[args.workload]
    A, eps1 = W.A(), W.eps1()
    masks = W.masks()
    kp = W.kpoints()
    nk = len(kp)
    ctxs = [api.pc_create(A, W.n, eps1, masks, device=local) for _ in range(max(1, args.streams))]
    for c_ in ctxs:
        if args.guard is not None:
            api.pc_set_option(c_, "guard", args.guard)
        if args.w_guard is not None:
            api.pc_set_option(c_, "w_guard", args.w_guard)
        api.pc_set_option(c_, "precond", 1 if args.precond == "eps" else 0)
    ctx = ctxs[0]

    def kidx(s, r=None):
        r = rank if r is None else r
        if args.warm_start:  # contiguous stretch per rank
            return (r * (args.warmup + args.steps + len(ctxs)) + s) % nk
        return (r + world * s) % nk

    def run(svals):
        """Solve a step set.  Cold start: the public band_structure call -- the k-points of ALL ranks
        (the union of every rank's idx_list) go into one dynamic queue (atomic counter in the process
        group's store), each rank's contexts draw from it, one all-gather returns every result; this
        rank's rows (k-points kidx(s) of the step numbers svals) are returned in step order.  Warm start: contiguous stretches per rank."""
        svals = list(svals)
        idx_list = [kidx(s_) for s_ in svals]
        if args.warm_start:
            return bands.solve_warm(ctxs, kp, idx_list, W.nev, args.tol, args.maxit, 0)
        ks = sorted({kidx(s_, r) for r in range(world) for s_ in svals})
        res = bands.band_structure(ctxs, kp, nev=W.nev, tol=args.tol, maxit=args.maxit, seed=0,
                                   device=cdev, ks=ks, kbatch=args.kbatch)
        sel = np.array(idx_list, dtype=np.int64)
        return res["omega2"][sel], res["resid"][sel], res["iters"][sel], res["status"][sel]

    # warm-up: W solves (at least one per context: allocations, first touch, kernel attributes)
    nwarm = max(args.warmup, len(ctxs))
    wit = [int(v) for v in run(range(nwarm))[2]]
    for c_ in ctxs:  # launch counts only: per-class CUDA events would add event records and host waits
        api.pc_stats(c_, reset=True)
        api.pc_set_option(c_, "profile", 0)
    clk = Clocks(local)
    barrier()
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    svals = list(range(nwarm, nwarm + args.steps))
    idx = [kidx(s) for s in svals]
    e0.record()
    om, rs, it_, st_ = run(svals)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clocks = clk.stop()
    barrier()
    stats = None
    for c_ in ctxs:
        s_ = api.pc_stats(c_)
        api.pc_set_option(c_, "profile", 0)
        if stats is None:
            stats = s_
        else:
            for k_, v_ in s_.items():
                if isinstance(v_, dict):
                    for f_ in v_:
                        stats[k_][f_] += v_[f_]
                else:
                    stats[k_] += v_
    t = torch.tensor([ms], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * args.steps / (ms_max / 1000.0)
    res = [(om[i:i + 1], rs[i:i + 1], it_[i:i + 1], st_[i:i + 1]) for i in range(len(idx))]
    iters = [int(r[2][0]) for r in res]
    status = [int(r[3][0]) for r in res]
    # the one collective of the method (all-gather of omega^2, Res, iterations, status) ran
    # inside the timed band_structure call: world * steps rows
    gathered = world * args.steps if (world > 1 and not args.warm_start) else None

    # ---- the same timed steps with the other preconditioner (same k-points, same protocol), reported
    # under alt_precond: the headline stays on the paper's K_P^{-1} unless --precond eps
    alt = None
    if not args.no_alt and not args.warm_start:
        other = "eps" if args.precond == "kp" else "kp"
        for c_ in ctxs:
            api.pc_set_option(c_, "precond", 1 if other == "eps" else 0)
        run(range(len(ctxs)))  # one untimed solve per context
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        aom, ars, ait, ast = run(svals)
        a1.record()
        torch.cuda.synchronize()
        ta = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(ta, op=dist.ReduceOp.MAX)
        barrier()
        for c_ in ctxs:
            api.pc_set_option(c_, "precond", 1 if args.precond == "eps" else 0)
        alt = {"precond": PRECOND_DESC[other], "value": world * args.steps / (float(ta.item()) / 1000.0),
               "unit": "k-points/s", "ms_per_step": float(ta.item()) / args.steps,
               "iters": [int(v) for v in ait], "status": [int(v) for v in ast],
               "max_rel_diff_omega2_vs_headline": float(np.max(np.abs(aom - om) / np.abs(om))),
               "note": "same k-points and protocol as the headline steps, timed right after them"}

    # ---- pc_apply bandwidth (second half of the metric): a b-column block at n=128
    ncol = args.apply_cols
    X = torch.randn(ncol, 3 * W.n ** 3, dtype=torch.complex128, device=dev)
    Y = torch.empty_like(X)
    kk = kp[kidx(0)]
    for _ in range(3):
        api.pc_apply(ctx, kk, X, Y)
    api.pc_stats(ctx, reset=True)
    api.pc_set_option(ctx, "profile", 1)
    torch.cuda.synchronize()
    reps = 5
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(reps):
        api.pc_apply(ctx, kk, X, Y)
    a1.record()
    torch.cuda.synchronize()
    apply_ms = a0.elapsed_time(a1) / reps
    astats = api.pc_stats(ctx)
    api.pc_set_option(ctx, "profile", 0)
    hbm, hbm_src, fp64, fp64_src = peaks()
    pts = W.n ** 3 * ncol
    alg_gbs = 336.0 * pts / (apply_ms * 1e6)
    # design traffic of the 5-pass fused pipeline used for this medium (eps_13 = eps_23 = 0): z+K_A^H,
    # y, x-DFT+M_eps+x-DFT (+1 B mask), y, z+K_A+gamma K_B (re-reads x^) = 4 x 96 + 144 + 1 B/pt
    design_b = 513.0  # 5 passes: 96+16, 96, 97, 96, 96+16 B per point per column
    design_gbs = design_b * pts / (apply_ms * 1e6)
    apply = {"cols": ncol, "ms": apply_ms, "alg_bytes_per_point_col": 336,
             "alg_gbs": alg_gbs, "frac_of_8tbs": alg_gbs / 8000.0, "frac_of_measured_hbm": alg_gbs / hbm,
             "design_bytes_per_point_col": design_b, "design_gbs": design_gbs,
             "kernels": {k: {"ms_per_apply": v["ms"] / reps, "gbs": (v["bytes"] / v["ms"] / 1e6) if v["ms"] else None}
                         for k, v in astats.items() if isinstance(v, dict) and v["count"]}}
    # library composition of the same apply (cuFFT via torch.fft + elementwise torch kernels: the
    # paper's GPU recipe on this GPU); same input block, agreement checked
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from library_apply import LibraryApply
        lib_ap = LibraryApply(W.n, A, kk, eps1, masks, api.pc_gamma(ctx, kk), dev)
        Yl = lib_ap(X)
        rel = float(torch.linalg.vector_norm(Yl - Y) / torch.linalg.vector_norm(Y))
        torch.cuda.synchronize()
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0.record()
        for _ in range(reps):
            Yl = lib_ap(X)
        l1.record()
        torch.cuda.synchronize()
        lib_ms = l0.elapsed_time(l1) / reps
        apply["library_baseline"] = {"what": "torch.fft (cuFFT Z2Z 3-D, batch 3 x cols) + torch elementwise/roll "
                                             "kernels for kappa products and the CrossDoF stencil",
                                     "ms": lib_ms, "alg_gbs": 336.0 * pts / (lib_ms * 1e6),
                                     "speedup_fused": lib_ms / apply_ms, "rel_diff_vs_pc_apply": rel}
        del Yl, lib_ap
    except Exception as ex:  # pragma: no cover - report, never fall back
        apply["library_baseline"] = {"error": str(ex)[:200]}
    del X, Y
    torch.cuda.empty_cache()

    # ---- roofline of the dominant kernel class.  Inside the timed region the concurrent contexts'
    # kernels interleave, so a class's event time there includes the other streams' kernels; the
    # per-kernel durations come from one profiled solve of the first timed k-point on one context
    # (same k, same seed, nothing else on the GPU), the shares from the timed region.
    k0 = idx[0]
    api.pc_set_option(ctx, "kindex_offset", k0)
    api.pc_stats(ctx, reset=True)
    api.pc_set_option(ctx, "profile", 1)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    solo = api.pc_bands(ctx, kp[k0:k0 + 1], nev=W.nev, tol=args.tol, maxit=args.maxit)
    s1.record()
    torch.cuda.synchronize()
    solo_ms = s0.elapsed_time(s1)
    pst = api.pc_stats(ctx)
    api.pc_set_option(ctx, "profile", 0)
    api.pc_set_option(ctx, "kindex_offset", 0)
    pcls = {k: v for k, v in pst.items() if isinstance(v, dict) and v["ms"] > 0}
    dom = max(pcls, key=lambda k: pcls[k]["ms"])
    d = pcls[dom]
    traffic = load_json(os.path.join(ROOT, "profiles", "traffic.json"), {}) or {}
    ridge = fp64 * 1e3 / hbm  # flop per byte
    inten = d["flops"] / d["bytes"] if d["bytes"] else float("inf")
    if inten >= ridge:
        ach = d["flops"] / (d["ms"] * 1e9)
        roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": fp64, "unit": "TFLOP/s",
                "frac": ach / fp64, "peak_source": fp64_src,
                "dtype": "fp64 (DMMA m8n8k4; algorithmic 8 flop per complex MAC)"}
    else:
        ach = d["bytes"] / (d["ms"] * 1e6)
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "peak_source": hbm_src}
    roof["intensity_flop_per_byte"] = inten
    roof["ridge_flop_per_byte"] = ridge
    roof["traffic"] = traffic.get(dom)
    roof["share_of_step"] = d["ms"] / solo_ms
    roof["avg_launch_group_ms"] = d["ms"] / max(1, d["count"])
    roof["measured_over"] = (f"one profiled solve of timed k-point {k0} on one context ({int(solo['iters'][0])} "
                             f"iterations, {solo_ms:.1f} ms), CUDA events on the launching stream")
    roof["classes_solo"] = {k: {"ms": v["ms"], "share": v["ms"] / solo_ms,
                                "tflops": v["flops"] / (v["ms"] * 1e9),
                                "gbs": v["bytes"] / (v["ms"] * 1e6)} for k, v in pcls.items()}

    # ---- end to end through the public API with host buffers (rank-local): a band-structure job as a
    # user runs it -- contexts created from pinned host masks (upload included), the k-points solved by
    # bands.solve_concurrent (host k in, host omega^2 / Res out), contexts destroyed -- all timed.
    e2e = None
    if args.e2e_steps > 0:
        # the timed contexts are done: free them first (at C5 one context holds ~94 GB of the 180)
        for c_ in ctxs:
            c_.close()
        pin =torch.from_numpy(masks.reshape(-1)).pin_memory()
        pinned_masks = pin.numpy().reshape(masks.shape)
        nctx = len(ctxs)

        def e2e_job(svals):
            idx_list = [kidx(s_) for s_ in svals]
            ce = [api.pc_create(A, W.n, eps1, pinned_masks, device=local) for _ in range(nctx)]
            for c_ in ce:
                if args.guard is not None:
                    api.pc_set_option(c_, "guard", args.guard)
                if args.w_guard is not None:
                    api.pc_set_option(c_, "w_guard", args.w_guard)
                api.pc_set_option(c_, "precond", 1 if args.precond == "eps" else 0)
            res = bands.band_structure(ce, kp, nev=W.nev, tol=args.tol, maxit=args.maxit, seed=0, device=cdev,
                                       ks=sorted({kidx(s_, r) for r in range(world) for s_ in svals}),
                                       kbatch=args.kbatch)
            sel = np.array(idx_list, dtype=np.int64)
            out = (res["omega2"][sel], res["resid"][sel], res["iters"][sel], res["status"][sel])
            for c_ in ce:
                c_.close()
            return out

        # one untimed job: steady state (the library caches the workspace of a destroyed context for
        # the next one on the device, see pc_destroy / pc_trim)
        e2e_job([0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # the same k-points as the timed device steps (when e2e_steps == steps), so E and value differ only
        # by what the end-to-end path adds (uploads, context setup, host round trips)
        e_it = [int(v) for v in e2e_job(range(nwarm, nwarm + args.e2e_steps))[2]]
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        tt = torch.tensor([te], dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        b = W.nev + (args.guard if args.guard is not None else 6)
        # per context: packed indicator masks (1 B/point) + twiddles and symbol tables; per k: 24 B k-point
        h2d = (nctx * (W.n ** 3 + 16 * W.n)) / args.e2e_steps + 24
        d2h = int(np.mean(e_it)) * (2 * b * 8 + 8) + b * 8
        e2e = {"value": world * args.e2e_steps / float(tt.item()), "unit": "k-points/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "iters": e_it,
               "note": f"one job of {args.e2e_steps} k-points per rank: pc_create x {nctx} from pinned host masks "
                       "(upload included) + bands.band_structure (dynamic k queue, concurrent contexts, one all-gather) "
                       "with host k-points and host omega^2/Res outputs + pc_destroy, wall clock"}

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = oracle_baseline(args, W, idx, with_c2=args.cpu_c2)
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "error": str(ex)[:300]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "k-points/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(W, args), "kpoints_per_rank": args.steps,
                "parallelism": (f"k-path over {world} GPU(s) from one dynamic queue, {len(ctxs)} concurrent "
                                f"k-point solve(s) per GPU, one all-gather"
                                if world <= torch.cuda.device_count() else
                                f"functional check: {world} ranks sharing {torch.cuda.device_count()} GPU(s) "
                                f"({args.dist_backend}), one dynamic queue, {len(ctxs)} concurrent k-point solve(s) "
                                f"per rank, one all-gather -- not a scaling result"),
                "iters": iters, "status": status, "warmup_iters": wit, "alt_precond": alt,
                "omega2_first_k": om[0].tolist(), "resid_max": float(rs.max()),
                "apply": apply, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": stats["launches"], "clocks": clocks,
                "algorithmic_timed_region": {k: {"gflop": v["flops"] / 1e9, "gbytes": v["bytes"] / 1e9}
                                             for k, v in stats.items() if isinstance(v, dict) and v["bytes"] > 0},
                "gathered_rows": gathered}
        print(json.dumps(line), flush=True)
    for c_ in ctxs:
        c_.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
