"""Host setup (pcg_plan_build: validation, anchor check, AINV, Z / Z^T packing) wall time per
config, best of N builds; PCG_VERBOSE=1 prints the stages.  Usage: plan_time.py cfg4 [cfg5] [-n 3]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("-")]
n = int(sys.argv[sys.argv.index("-n") + 1]) if "-n" in sys.argv else 3
for name in [a for a in args if a.startswith("cfg")] or ["cfg4"]:
    p = synth.config(name)
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        P = pcg.Plan(p.cE, p.cN, p.mask, tau=0.1)
        ts.append(time.perf_counter() - t)
        P.close()
    print(f"{name} plan: best {min(ts):.3f} s, all {' '.join(f'{x:.3f}' for x in ts)}", flush=True)
