"""Iterations per rank count P for block-local AINV (w = 0) and halo-AINV (w > 0), run through the
multi-rank device path on one GPU (pcg_solve_local_ranks: P contexts, device-copy exchanges).
Times are of that one-GPU emulation (ranks' phases serialised on one stream), NOT multi-GPU times.

    python tools/multirank_modes.py --configs cfg2,cfg3,cfg4 --ranks 1,2,4,8 --halos 0,3
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="cfg2,cfg3,cfg4")
ap.add_argument("--ranks", default="1,2,4,8")
ap.add_argument("--halos", default="0,3")
ap.add_argument("--tol", type=float, default=1e-10)
a = ap.parse_args()
for name in a.configs.split(","):
    p = synth.config(name)
    S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1)
    b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
    S.close()
    for P in (int(x) for x in a.ranks.split(",")):
        for w in (int(x) for x in a.halos.split(",")):
            if P == 1 and w > 0:
                continue
            t0 = time.perf_counter()
            R = pcg.LocalRanks(p.cE, p.cN, p.mask, P, tau=0.1, ainv_halo=w)
            setup = time.perf_counter() - t0
            R.solve(b, tol=a.tol, maxit=200000)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, k, hist, rep = R.solve(b, tol=a.tol, maxit=200000)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(json.dumps({"config": name, "P": P, "ainv_halo": w, "iterations": k, "converged": rep["converged"],
                              "true_rel_residual": rep["true_rel_residual"], "setup_wall_s": setup,
                              "emulated_solve_ms": dt * 1e3, "emulated_us_per_iter": dt / k * 1e6}), flush=True)
            R.close()
