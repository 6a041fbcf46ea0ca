"""Block timeline of one PCG iteration (diagnostic build with -DPCG_TIMELINE).

    python -m paper_1210_1878_b200.build --variant tl PCG_TIMELINE
    PCG_LIB=paper_1210_1878_b200/_build/tl/libpcg.so python tools/timeline.py --config cfg4
Runs a graph solve with tol 0 and an even maxit (so the last K1/K2/K3 launches are live), then
prints, per kernel, the spread of block entry / post-wait / loop-end times and the last block's
finish, relative to the earliest K1 entry (microseconds)."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--maxit", type=int, default=200)
a = ap.parse_args()
p = synth.config(a.config)
S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1)
b = S.apply_operator(torch.from_numpy(synth.xstar(p)).cuda())
lib = ctypes.CDLL(os.environ["PCG_LIB"])
S.solve(b, tol=0.0, maxit=a.maxit)
torch.cuda.synchronize()
units = np.zeros(2048, dtype=np.uint32)
lib.pcg_diag_units(units.ctypes.data_as(ctypes.c_void_p), 1)
S.solve(b, tol=0.0, maxit=a.maxit)
torch.cuda.synchronize()
lib.pcg_diag_units(units.ctypes.data_as(ctypes.c_void_p), 0)
buf = np.zeros((3, 2048, 8), dtype=np.uint64)
assert lib.pcg_diag_timeline(buf.ctypes.data_as(ctypes.c_void_p)) == 0
grid = [S._grid_sizes[i] if hasattr(S, "_grid_sizes") else None for i in range(3)]
t0 = min(int(v) for v in buf[0, :, 0] if v > 0)
for kk, name in enumerate(("K1", "K2", "K3")):
    T = buf[kk].astype(np.int64)
    live = T[:, 0] > 0
    T = T[live]
    rel = (T - t0) / 1e3
    def q(c):
        v = rel[:, c][T[:, c] > 0]
        return "min %7.2f  p50 %7.2f  max %7.2f" % (v.min(), np.median(v), v.max()) if len(v) else "-"
    fin = rel[:, 3][T[:, 3] > 0]
    print(f"{name} blocks={live.sum():4d} entry[{q(0)}] wait[{q(1)}] loopend[{q(2)}] last_done={fin.max() if len(fin) else float('nan'):7.2f}")
    busy = (rel[:, 2] - rel[:, 1])
    print(f"    block busy (loopend-wait): mean {busy.mean():6.2f} min {busy.min():6.2f} max {busy.max():6.2f}")
    idx = np.nonzero(live)[0]
    slow = np.argsort(-rel[:, 2])[:5]
    print("    slowest blocks (id, wait, loopend):", [(int(idx[s]), round(float(rel[s, 1]), 2), round(float(rel[s, 2]), 2)) for s in slow])
nz = units[units > 0] / (2 * a.maxit)
print("units per block per K2+K3 launch (all dynamic kernels, summed / launches): mean %.2f min %.2f max %.2f" % (nz.mean(), nz.min(), nz.max()))
print("blocks with most units:", [(int(i), round(float(units[i]) / (2 * a.maxit), 2)) for i in np.argsort(-units)[:5]])

tail = np.zeros((3, 4), dtype=np.uint64)
if hasattr(lib, "pcg_diag_tail"):
    lib.pcg_diag_tail(tail.ctypes.data_as(ctypes.c_void_p))
    for kk in range(3):
        if tail[kk, 0]:
            lb = int(np.argmax(buf[kk, :, 3]))
            if tail[kk, 2] and tail[kk, 3]:
                print("K%d fin: sums->before set_cond %.2f us, set_cond %.2f us, after set_cond -> block end %.2f us" % (
                      kk + 1, (int(tail[kk, 2]) - int(tail[kk, 1])) / 1e3, (int(tail[kk, 3]) - int(tail[kk, 2])) / 1e3,
                      (int(buf[kk, :, 3].max()) - int(tail[kk, 3])) / 1e3))
            print("K%d last block %d: loopend->counted %.2f us, count->sums %.2f us, sums->end %.2f us; latest loopend of any block -> its loopend %.2f us" % (
                  kk + 1, lb, (int(tail[kk, 0]) - int(buf[kk, lb, 2])) / 1e3, (int(tail[kk, 1]) - int(tail[kk, 0])) / 1e3,
                  (int(buf[kk, :, 3].max()) - int(tail[kk, 1])) / 1e3, (int(buf[kk, lb, 2]) - int(buf[kk, :, 2].max())) / 1e3))

for kk in (1, 2):
    T = buf[kk].astype(np.int64)
    live = T[:, 0] > 0
    if not (T[live, 4] > 0).any():
        continue
    ids = np.nonzero(live)[0]
    rel = (T[live] - t0) / 1e3
    stat = rel[:, 4] - rel[:, 1]
    order = np.argsort(-rel[:, 2])[:8]
    print("K%d static phase: mean %.2f min %.2f max %.2f us; dynamic units/block mean %.2f" % (kk + 1, stat.mean(), stat.min(), stat.max(), T[live, 6].mean()))
    for o in order:
        print("   block %4d static %.2f us (%d units) + dyn %d units -> loopend %.2f" % (ids[o], stat[o], T[live][o, 7], T[live][o, 6], rel[o, 2]))
