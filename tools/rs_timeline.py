"""Per-pass durations of the resident-strip loop (diagnostic build -DRS_TIMELINE, GPU box).
   python -m paper_1210_1878_b200.build --variant rstl RS_TIMELINE
   PCG_LIB=paper_1210_1878_b200/_build/rstl/libpcg.so python tools/rs_timeline.py cfg4 ainv"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

NAMES = ["top", "1a d", "1b stencil+part", "barrier1", "final1", "2A r", "2B Zt", "flag", "2C t",
         "2D Z+part", "barrier2", "final2"]
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
precond = sys.argv[2] if len(sys.argv) > 2 else "ainv"
p = synth.config(name)
S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, precond=precond, device=0)
b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
L = pcg.lib()
L.pcg_rs_timeline.argtypes = [C.c_void_p, C.c_void_p]
buf = np.zeros((160, 12), dtype=np.uint64)
S.solve(b, tol=1e-10)
L.pcg_rs_timeline(S._h, buf.ctypes.data)          # reset
x, k, h, rep = S.solve(b, tol=1e-10)
assert L.pcg_rs_timeline(S._h, buf.ctypes.data) == 1
nb = 148
t = buf[:nb].astype(np.float64) / k / 1e3          # us per iteration
print(f"{name} {precond}: {k} iterations, {rep['solve_s'] / k * 1e6:.2f} us/iteration")
for s_, n_ in enumerate(NAMES):
    col = t[:, s_]
    print(f"  {n_:16s} mean {col.mean():7.2f}  max {col.max():7.2f}  min {col.min():7.2f}  argmax {int(col.argmax())}")
print(f"  {'sum':16s} mean {t.sum(1).mean():7.2f}")
