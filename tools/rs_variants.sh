#!/bin/bash
# time the resident-strip build variants (tools/rs_check.py with PCG_LIB) on one box
for v in "$@"; do
  echo "== $v"
  PCG_LIB=paper_1210_1878_b200/_build/$v/libpcg.so timeout 90 python tools/rs_check.py cfg4 2>&1 | grep -v "structured Z" | tail -4
done
