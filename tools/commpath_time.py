import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch, paper_1210_1878_b200 as pcg
from paper_1210_1878_b200 import synth
p = synth.config(sys.argv[1])
S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1, comm_path=True)
b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
for _ in range(2): S.solve(b, tol=1e-10)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(3): x, k, h, r = S.solve(b, tol=1e-10)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
print(json.dumps({"cfg": sys.argv[1], "multi_graph": os.environ.get("PCG_MULTI_GRAPH", "0"), "its": k, "ms": dt * 1e3, "us_per_it": dt * 1e6 / k}))
S.close()
