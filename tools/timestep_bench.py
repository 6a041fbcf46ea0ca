"""Time-stepping driver at a BASELINE config: one setup, N time steps of
pcg_solve with NEMO's first guess, against cold solves.  One JSON line per warm mode.

    python tools/timestep_bench.py [--config cfg4] [--steps 30] [--tol 1e-10]
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
from paper_1210_1878_b200 import synth, timestep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--tol", type=float, default=1e-10)
ap.add_argument("--tau", type=float, default=0.1)
a = ap.parse_args()
p = synth.config(a.config)
t0 = time.perf_counter()
S = pcg.Solver(p.cE, p.cN, p.mask, tau=a.tau)
setup_s = time.perf_counter() - t0
series = [torch.from_numpy(f).cuda() for f in synth.forcing_series(p, a.steps)]
rhs = [S.apply_operator(f) for f in series]               # b^n = A D*(t_n) through the library
for warm in timestep.WARM:
    st = timestep.Stepper(S, warm)
    its, errs = [], []
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for n in range(a.steps):
        x, k, rep = st.step(rhs[n], tol=a.tol, maxit=20 * p.ni * p.nj)
        its.append(k)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    errs = float(max(((x - series[-1]).norm() / series[-1].norm()).item(), 0.0))
    print(json.dumps({"config": a.config, "warm": warm, "steps": a.steps, "tol": a.tol, "setup_s": setup_s,
                      "iterations": its, "mean_iterations": float(np.mean(its)),
                      "mean_iterations_after_2": float(np.mean(its[2:])) if len(its) > 2 else None,
                      "ms_total": ms, "ms_per_step": ms / a.steps, "last_step_err_vs_target": errs}), flush=True)
S.close()
