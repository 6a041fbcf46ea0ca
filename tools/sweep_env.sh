#!/bin/bash
# usage: tools/sweep_env.sh <variant> "<ENV=..> <ENV=..>" ...   (cfg4, K1 rows 4)
v=$1; shift
for envs in "$@"; do
  echo "== $v $envs"
  env $envs PCG_LIB=paper_1210_1878_b200/_build/$v/libpcg.so timeout 120 python tools/tune_rows.py --config ${CFG:-cfg4} --rows 4 2>&1 | grep "^{"
done
