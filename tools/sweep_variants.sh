#!/bin/bash
# Sweep tuning variants built with `python -m paper_1210_1878_b200.build --variant <name> -D...`
cfg=${CFG:-cfg4}; SR=${SR:-1,2,4}
for v in "$@"; do
  echo "== variant $v"
  PCG_LIB=paper_1210_1878_b200/_build/$v/libpcg.so timeout 300 python tools/tune_rows.py --config $cfg --rows 4 --sell-rows $SR 2>&1 | grep "^{"
done
