"""pcg_setup wall time and the plan's stages (PCG_VERBOSE) through the Solver, per config (GPU box).
Usage: setup_time.py cfg4 [cfg5]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

for name in sys.argv[1:] or ["cfg4"]:
    p = synth.config(name)
    for _ in range(2):
        t = time.perf_counter()
        S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1, device=0)
        wall = time.perf_counter() - t
        b = S.apply_operator(torch.ones(p.mask.shape, dtype=torch.float64, device="cuda"))
        _, _, _, rep = S.solve(b, tol=1e-10, maxit=1)
        print(f"{name}: setup_s {rep['setup_s']:.3f}, Solver() wall {wall:.3f} s", flush=True)
        S.close()
