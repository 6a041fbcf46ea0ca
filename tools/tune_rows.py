"""Sweep the rows-per-block tile height (PCG_ROWS_PER_BLOCK) and report per-kernel times.

    python tools/tune_rows.py --config cfg4 --rows 1,2,4,8,16
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--rows", default="1,2,4,8,16")
ap.add_argument("--sell-rows", default="")
ap.add_argument("--win", default="")
ap.add_argument("--precond", default="ainv")
ap.add_argument("--iters", type=int, default=60)
a = ap.parse_args()
p = synth.config(a.config)
xs = torch.from_numpy(synth.xstar(p)).cuda()
out = []
combos = [(int(r), None) for r in a.rows.split(",")] if not a.sell_rows else \
    [(int(r), int(s)) for r in a.rows.split(",") for s in a.sell_rows.split(",")]
wins = [int(w) for w in a.win.split(",")] if a.win else [None]
combos = [(R, SR, W) for (R, SR) in combos for W in wins]
for R, SR, WN in combos:
    if WN is not None:
        os.environ["PCG_WIN"] = str(WN)
    os.environ["PCG_ROWS_PER_BLOCK"] = str(R)
    if SR is not None:
        os.environ["PCG_SELL_ROWS"] = str(SR)
    S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1, precond=a.precond)
    b = S.apply_operator(xs)
    for _ in range(2):
        x, k, hist, rep = S.solve(b, tol=1e-10, maxit=100000)
    ts = []
    for _ in range(3):
        x, k, hist, rep = S.solve(b, tol=1e-10, maxit=100000)
        ts.append(rep["solve_s"])
    ms, by = S.kernel_times(a.iters)
    r = {"rows": S.tile_rows, "sell_rows": SR, "win": WN, "iters": k, "solve_ms": 1e3 * min(ts), "us_per_iter": 1e6 * min(ts) / k,
         "K1_us": 1e3 * ms[0], "K2_us": 1e3 * ms[1], "K3_us": 1e3 * ms[2], "iter_us_events": 1e3 * ms[3],
         "K_GBps": [float(by[i] / (ms[i] * 1e-3) / 1e9) if ms[i] > 0 else None for i in range(3)]}
    print(json.dumps(r), flush=True)
    out.append(r)
    S.close()
