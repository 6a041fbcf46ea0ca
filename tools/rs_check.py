"""Resident-strip driver vs the three-kernel graph: bitwise equality and timings (GPU box)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402


def run(p, b, precond, rs, reps=3, tol=1e-10):
    os.environ["PCG_RS"] = "1" if rs else "0"
    S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, precond=precond, device=0)
    x, k, h, rep = S.solve(b, tol=tol)
    ts = []
    for _ in range(reps):
        x, k, h, rep = S.solve(b, tol=tol)
        ts.append(rep["solve_s"])
    lt = S.loop_time()
    S.close()
    return x.cpu().numpy(), k, h, min(ts), lt


cfgs = sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]
for name in cfgs:
    p = synth.config(name)
    xs = synth.xstar(p)
    S0 = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1, device=0)
    b = S0.apply_operator(torch.from_numpy(xs).cuda())
    S0.close()
    for precond in ("ainv", "jacobi"):
        x0, k0, h0, t0, _ = run(p, b, precond, False)
        x1, k1, h1, t1, lt = run(p, b, precond, True)
        same = k0 == k1 and np.array_equal(h0, h1) and np.array_equal(x0, x1)
        print(f"{name} {precond}: graph {k0} it {t0*1e3:.3f} ms ({t0/k0*1e6:.2f} us/it) | rs {k1} it {t1*1e3:.3f} ms "
              f"({t1/max(k1,1)*1e6:.2f} us/it) loop {lt[0]:.3f} ms / {lt[1]} it | bitwise={same}", flush=True)
        if not same:
            d = np.abs(x0 - x1).max()
            print(f"   maxdiff x {d:.3e}  hist0 {h0[:4]} hist1 {h1[:4]}")
