"""Per-kernel times (host-loop CUDA events, pcg_kernel_times) of K1/K2/K3 on one config; run with
PCG_LIB=<variant build> to compare kernel forms.  Usage: k1_time.py [cfg5] [iterations]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = synth.config(name)
S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, device=0)
b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
x, k, h, rep = S.solve(b, tol=1e-12, maxit=40)
ms, by = S.kernel_times(n)
print(os.environ.get("PCG_LIB", "default"), name, "K1 %.1f us (%.0f GB/s)  K2 %.1f  K3 %.1f" % (
    ms[0] * 1e3, by[0] / (ms[0] * 1e-3) / 1e9, ms[1] * 1e3, ms[2] * 1e3), flush=True)
S.close()
