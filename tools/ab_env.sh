#!/bin/bash
# A/B bench lines at cfg4 for env settings given one per argument (e.g. "PCG_SZ=0" "PCG_SZ=1 PCG_FUSE23=1").
# BENCH_ARGS adds bench.py flags. Lines -> gpurun_out/ab_env.jsonl, summary on stdout.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/ab_env.jsonl; : > $out
for setting in "$@"; do
  echo "== $setting" >> gpurun_out/ab_env.log
  line=$(env $setting timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu ${BENCH_ARGS} 2>>gpurun_out/ab_env.log | tail -n 1)
  SETTING="$setting" LINE="$line" python -c 'import json,os; print(json.dumps({"env": os.environ["SETTING"], "line": json.loads(os.environ["LINE"] or "null")}))' >> $out
done
python - <<'PY'
import json
for l in open("gpurun_out/ab_env.jsonl"):
    d = json.loads(l); L = d["line"]
    if not L:
        print(d["env"], "| FAILED"); continue
    c = L["config"]
    ks = {k: (round(v["ms"] * 1e3, 1) if isinstance(v, dict) else round(v * 1e3, 1)) for k, v in c["kernels"].items() if "GBps" not in k}
    print(d["env"], "| iter/s", round(L["value"]), "| ms", round(L["ms_per_step"], 2), "| its", c["iterations_per_solve"][0],
          "| us/it", round(1e3 * L["ms_per_step"] / c["iterations_per_solve"][0], 2), "|", ks, "| frac", round(L["roofline"]["frac"], 3))
PY
