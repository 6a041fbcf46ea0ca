"""Small driver for ncu / sanitizer runs: set up a config and run one solve.

    python tools/prof_run.py --config cfg4 --maxit 20 [--precond ainv] [--solves 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--maxit", type=int, default=20)
ap.add_argument("--tol", type=float, default=0.0)
ap.add_argument("--precond", default="ainv")
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
p = synth.config(a.config)
S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1, precond=a.precond, flags=a.flags)
b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
for _ in range(a.solves):
    x, k, hist, rep = S.solve(b, tol=a.tol, maxit=a.maxit)
torch.cuda.synchronize()
print(f"{a.config} {a.precond}: {k} iterations, relres {hist[-1]:.3e}, solve {rep['solve_s']*1e3:.3f} ms")
S.close()
