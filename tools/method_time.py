"""Time one solve of each PCG form (Alg. 1 default driver, Chronopoulos-Gear, pipelined) on a
config: iterations, solve seconds, microseconds per iteration.  Usage: method_time.py cfg4 [tol]"""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_1210_1878_b200 as pcg
from paper_1210_1878_b200 import synth

name = sys.argv[1]
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-10
p = synth.config(name)
for label, flags in (("alg1", 0), ("cg1", pcg.FLAG_SINGLE_REDUCTION), ("pipe", pcg.FLAG_PIPELINED)):
    S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, flags=flags, device=0)
    b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
    best = None
    for _ in range(3):
        x, k, h, rep = S.solve(b, tol=tol)
        best = rep["solve_s"] if best is None else min(best, rep["solve_s"])
    print(f"{name} {label:5s} driver={rep.get('driver_name', rep.get('driver'))} k={k} solve_s={best:.4f} "
          f"us/it={1e6 * best / max(k, 1):.1f} true_rel={rep['true_rel_residual']:.3e}", flush=True)
    S.close()
