"""One rank through the NCCL path (PCG_FLAG_COMM_PATH): iterations and time per iteration.
    [CG1=1] [PCG_MULTI_GRAPH=0] python tools/commpath_time.py cfg4
"""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch, paper_1210_1878_b200 as pcg
from paper_1210_1878_b200 import synth
p = synth.config(sys.argv[1])
S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1, comm_path=True,
               flags=pcg.FLAG_SINGLE_REDUCTION if os.environ.get("CG1") == "1" else 0)
b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
for _ in range(2): S.solve(b, tol=1e-10)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(3): x, k, h, r = S.solve(b, tol=1e-10)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
print(json.dumps({"cfg": sys.argv[1], "method": "cg1" if os.environ.get("CG1") == "1" else "pcg", "multi_graph": os.environ.get("PCG_MULTI_GRAPH", "1"), "its": k, "ms": dt * 1e3, "us_per_it": dt * 1e6 / k}))
S.close()
