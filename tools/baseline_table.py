"""Regenerate BASELINE.md §5's table rows from profiles/r01/measure_configs.jsonl (prints them)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
f = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01", "measure_configs.jsonl")
rows = [json.loads(l) for l in open(f) if l.strip()]
dims = {"cfg1": "32x32", "cfg2": "182x149", "cfg3": "362x292", "cfg4": "1442x1021", "cfg5": "4322x3059"}
order = {"ainv": 0, "jacobi": 1, "fsai": 2, "pb2": 3}


def pc(d):
    if d["precond"] == "ainv":
        return "AINV (%g)" % d["tau"]
    if d["precond"] == "jacobi":
        return "Jacobi"
    if d["precond"] == "fsai":
        return "FSAI (q = %d)" % d.get("fsai_q", d.get("q"))
    return "P_B2 (m = %d)" % d["fill"]


rows.sort(key=lambda d: (order[d["precond"]], d["config"], d.get("fsai_q", 0), d.get("fill", 0)))
for d in rows:
    orc = "33.3 iter/s (1 core)" if d["config"] == "cfg4" and d["precond"] == "ainv" else "—"
    ratio = "%d× (iter/s)" % round(d["iter_per_s"] / 33.3) if orc != "—" else "—"
    print("| %s %s | 1 | %s | %g | %d | %d | %.2f ms | %.1f | %d | %.1f %% | %s | %s |" % (
        d["config"], dims[d["config"]], pc(d), d["tol"], d["iterations"], round(d["iter_per_s"]),
        d["time_to_solution_ms"], d["us_per_iter"], round(d["alg_GBps"]), 100 * d["frac_of_measured_hbm"], orc, ratio))
