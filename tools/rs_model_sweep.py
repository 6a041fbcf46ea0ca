"""Sweep the resident-strip partition's cost model (PCG_RS_MODEL = K1 ocean chunk, K1 shared per
chunk, K2/K3 ocean chunk, per overflow round, K2/K3 shared per chunk; us) on one config: loop us
per iteration (best of 3 solves) for each model.  Usage: rs_model_sweep.py cfg4 ainv m1 m2 ..."""
import os
import subprocess
import sys

name, precond, models = sys.argv[1], sys.argv[2], sys.argv[3:]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = ("import sys, torch; sys.path.insert(0, %r); import paper_1210_1878_b200 as pcg; "
        "from paper_1210_1878_b200 import synth; p = synth.config(%r); "
        "S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, precond=%r, device=0); "
        "b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda()); best = 1e9\n"
        "for _ in range(3):\n"
        "    S.solve(b, tol=1e-10); lt = S.loop_time(); best = min(best, lt[0] / lt[1] * 1e3)\n"
        "print(best)" % (root, name, precond))
for m in models:
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=dict(os.environ, PCG_RS_MODEL=m))
    print(m, r.stdout.strip() or r.stderr[-300:], flush=True)
