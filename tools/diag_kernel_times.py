import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1210_1878_b200 as pcg
from paper_1210_1878_b200 import synth
p = synth.config("cfg4")
for sr in (1, 2):
    os.environ["PCG_SELL_ROWS"] = str(sr)
    S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1, flags=pcg.FLAG_HOST_LOOP)
    b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
    S.solve(b, tol=0.0, maxit=5)
    try:
        ms, by = S.kernel_times(60)
    except Exception as e:
        print("err", e); continue
    print(os.environ.get("PCG_LIB", "default")[-20:], sr, [round(1e3 * m, 1) for m in ms])
    S.close()
