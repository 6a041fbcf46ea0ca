"""Short resident-strip solve for ncu (cfg4, AINV(0.1), tol 0, N iterations after one warm solve)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
precond = sys.argv[3] if len(sys.argv) > 3 else "ainv"
p = synth.config(name)
S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, precond=precond, device=0)
b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
S.solve(b, tol=0.0, maxit=n)
x, k, h, rep = S.solve(b, tol=0.0, maxit=n)
torch.cuda.synchronize()
print(name, precond, k, rep["solve_s"] / k * 1e6, "us/it", S.loop_time())
