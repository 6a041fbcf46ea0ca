#!/bin/bash
# A/B of resident-strip build variants on one box: default build vs each variant, alternating,
# cfg4 AINV + Jacobi us per iteration (tools/rs_check.py).  Usage: rs_ab.sh v1 v2 ...
for round in 1 2; do
  echo "== default"; timeout 90 python tools/rs_check.py cfg4 2>&1 | grep -E "ainv|jacobi" | sed "s/.*| rs/rs/"
  for v in "$@"; do
    echo "== $v"; PCG_LIB=paper_1210_1878_b200/_build/$v/libpcg.so timeout 90 python tools/rs_check.py cfg4 2>&1 | grep -E "ainv|jacobi" | sed "s/.*| rs/rs/"
  done
done
