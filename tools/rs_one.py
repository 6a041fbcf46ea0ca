import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1210_1878_b200 as pcg
from paper_1210_1878_b200 import synth
name, precond = sys.argv[1], sys.argv[2]
p = synth.config(name)
S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, precond=precond, device=0)
b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
t = time.time()
print("solving", flush=True)
x, k, h, rep = S.solve(b, tol=1e-10)
print(name, precond, k, rep["solve_s"], S.loop_time(), time.time() - t, flush=True)
