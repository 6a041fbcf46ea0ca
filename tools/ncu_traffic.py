"""Turn an `ncu --set full` capture of K1/K2/K3 into profiles/ncu_traffic.json (roofline.traffic).

    ncu -i gpurun_out/full.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_traffic.py raw.csv --config cfg4 --source "<how it was captured>"
"""
import argparse
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {"k1_kernel": "K1_stencil", "k1_flat_kernel": "K1_stencil", "k2_ainv_kernel": "K2_ZTr", "k3_ainv_kernel": "K3_Zt",
         "k2_tma_kernel": "K2_ZTr", "k3_tma_kernel": "K3_Zt"}

ap = argparse.ArgumentParser()
ap.add_argument("raw")
ap.add_argument("--config", default="cfg4")
ap.add_argument("--source", default="")
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"))
a = ap.parse_args()
rows = list(csv.reader(open(a.raw)))
hdr, units = rows[0], dict(zip(rows[0], rows[1]))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "": 1.0, "cycle": 1.0, "register/thread": 1.0, "block": 1.0, "thread": 1.0}


def num(s, col=None):
    """value in base units (bytes, seconds) using the unit row of the raw page"""
    try:
        v = float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None
    return v * SCALE.get(units.get(col, ""), 1.0) if col else v


out, det = {}, {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    kname = d["Kernel Name"]
    key = next((v for k, v in NAMES.items() if k + "(" in kname or k + "<" in kname), None)
    if key is None or key in det:
        continue
    rd, wr = num(d["dram__bytes_read.sum"], "dram__bytes_read.sum"), num(d["dram__bytes_write.sum"], "dram__bytes_write.sum")
    dur = num(d["gpu__time_duration.sum"], "gpu__time_duration.sum")
    det[key] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "duration_us": dur * 1e6 if dur else None,
                "dram_GBps": (rd + wr) / dur / 1e9 if dur else None,
                "sm_active_frac": (num(d.get("sm__cycles_active.avg", "")) or 0) / (num(d.get("sm__cycles_elapsed.avg", "")) or 1),
                "registers": num(d.get("launch__registers_per_thread", "")), "grid": num(d.get("launch__grid_size", ""))}
    out[key] = rd + wr
res = {a.config: out, "_detail": det, "_source": a.source}
json.dump(res, open(a.out, "w"), indent=1)
print(json.dumps(res, indent=1))
