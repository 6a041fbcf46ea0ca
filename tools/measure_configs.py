"""Measure BASELINE.json's configs on one GPU: iterations, time-to-solution, iterations/s,
effective algorithmic bandwidth, for AINV(tau) and Jacobi.

    python tools/measure_configs.py [--configs cfg2,cfg3,cfg4,cfg5] [--taus 0.1] [--jacobi]
Prints one JSON object per run.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg4")
ap.add_argument("--taus", default="0.1")
ap.add_argument("--jacobi", action="store_true")
ap.add_argument("--fsai", default="", help="comma list of FSAI bandwidths q (the paper's preconditioner)")
ap.add_argument("--fill", default="", help="comma list of P_B2 fills m (AINV with tau = 0, m entries per column)")
ap.add_argument("--tol", type=float, default=None)
ap.add_argument("--cg1", action="store_true", help="Chronopoulos-Gear single-reduction PCG (NEXT-2)")
ap.add_argument("--pipe", action="store_true", help="pipelined PCG (NEXT-2)")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
TOL = {"cfg1": 1e-10, "cfg2": 1e-10, "cfg3": 1e-10, "cfg4": 1e-10, "cfg5": 1e-12}
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6650.0
for name in a.configs.split(","):
    t0 = time.perf_counter()
    p = synth.config(name)
    gen_s = time.perf_counter() - t0
    xs = torch.from_numpy(synth.xstar(p)).cuda()
    runs = [("ainv", float(t)) for t in a.taus.split(",") if t] + ([("jacobi", 0.0)] if a.jacobi else []) + \
        [("fsai", float(q)) for q in a.fsai.split(",") if q] + [("pb2", float(f)) for f in a.fill.split(",") if f]
    for pc, tau in runs:
        t0 = time.perf_counter()
        S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.0 if pc == "pb2" else (tau if pc != "fsai" else 0.1),
                       precond="ainv" if pc == "pb2" else pc, fsai_q=int(tau) if pc == "fsai" else 4,
                       ainv_fill=int(tau) if pc == "pb2" else 0,
                       flags=pcg.FLAG_SINGLE_REDUCTION if a.cg1 else pcg.FLAG_PIPELINED if a.pipe else 0)
        setup_wall = time.perf_counter() - t0
        b = S.apply_operator(xs)
        tol = a.tol if a.tol is not None else TOL[name]
        x, k, hist, rep = S.solve(b, tol=tol, maxit=200000)
        best = 1e9
        for _ in range(a.reps):
            x, k, hist, rep = S.solve(b, tol=tol, maxit=200000)
            best = min(best, rep["solve_s"])
        err = float(torch.linalg.norm(x - xs) / torch.linalg.norm(xs))
        bpi = rep["bytes_per_iter"]
        out = {"config": name, "grid": [p.ni, p.nj], "n_ocean": rep["n_ocean"], "precond": pc,
               "method": "cg1" if a.cg1 else "pipe" if a.pipe else "pcg",
               ({"fsai": "fsai_q", "pb2": "fill"}.get(pc, "tau")): (int(tau) if pc in ("fsai", "pb2") else tau), "tol": tol,
               "iterations": k, "converged": rep["converged"], "true_rel_residual": rep["true_rel_residual"],
               "err_vs_xstar": err, "time_to_solution_ms": best * 1e3, "iter_per_s": k / best,
               "us_per_iter": best / k * 1e6, "alg_bytes_per_iter_MB": bpi / 1e6,
               "alg_GBps": bpi * k / best / 1e9, "frac_of_measured_hbm": bpi * k / best / 1e9 / peak,
               "bytes_to_solution_GB": bpi * k / 1e9, "driver": rep.get("driver_name"),
               "z_per_col": rep["nnz_z"] / max(rep["n_ocean"], 1), "setup_s": rep["setup_s"],
               "setup_wall_s": setup_wall, "device_MB": S.device_bytes / 1e6, "gen_s": gen_s}
        print(json.dumps(out), flush=True)
        S.close()
