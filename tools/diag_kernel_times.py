"""Per-kernel CUDA-event times of the host-loop driver at a fixed iteration count (works for
diagnostic variants whose arithmetic no longer converges: PCG_DIAG=1 skips the iteration check).

    PCG_LIB=paper_1210_1878_b200/_build/<variant>/libpcg.so python tools/diag_kernel_times.py --config cfg4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PCG_DIAG", "1")
import torch  # noqa: E402

import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--iters", type=int, default=60)
a = ap.parse_args()
p = synth.config(a.config)
S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1, flags=pcg.FLAG_HOST_LOOP)
b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
S.solve(b, tol=0.0, maxit=5)
ms, by = S.kernel_times(a.iters)
print(os.environ.get("PCG_LIB", "default")[-28:], "K1/K2/K3/iter us:", [round(1e3 * m, 1) for m in ms])
S.close()
