"""Full CPU-oracle solves (the CPU baseline of SURVEY §8(d) / BASELINE.md §4) on this host:
setup (assembly + AINV) and solve seconds to tol, single thread (PLAIN order) and all cores
(CHUNKED order: OpenMP rows, fixed 4096-element chunk partials).  One JSON object per run.

    python tools/measure_oracle.py [--configs cfg1,cfg2,cfg3] [--chunked-only cfg4]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402
import bench  # noqa: E402  (cpu_info)

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="cfg1,cfg2,cfg3")
ap.add_argument("--chunked-only", default="", help="configs timed with all cores only")
ap.add_argument("--precond", default="ainv")
a = ap.parse_args()
TOL = {"cfg1": 1e-10, "cfg2": 1e-10, "cfg3": 1e-10, "cfg4": 1e-10, "cfg5": 1e-12}
cores, model = bench.cpu_info()
jobs = [(c, m) for c in a.configs.split(",") if c for m in ("plain", "chunked")] + \
       [(c, "chunked") for c in a.chunked_only.split(",") if c]
for name, mode in jobs:
    p = synth.config(name)
    t0 = time.perf_counter()
    A = oracle.assemble(p)
    M = oracle.ainv(A, 0.1 + 1e-9) if a.precond == "ainv" else None
    t1 = time.perf_counter()
    b = A.apply(A.from_grid(synth.xstar(p)))
    t2 = time.perf_counter()
    r = oracle.pcg(A, b, a.precond, M, TOL[name], maxit=A.n, mode=mode)
    t3 = time.perf_counter()
    print(json.dumps({"config": name, "precond": a.precond, "mode": mode, "threads": 1 if mode == "plain" else cores,
                      "cpu_model": model, "n_ocean": A.n, "tol": TOL[name], "iterations": r.iterations,
                      "converged": bool(r.converged), "setup_s": t1 - t0, "solve_s": t3 - t2,
                      "iter_per_s": r.iterations / (t3 - t2), "time_to_solution_s": (t1 - t0) + (t3 - t2)}), flush=True)
