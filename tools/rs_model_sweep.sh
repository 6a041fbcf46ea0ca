#!/bin/bash
# Sweep the resident-strip partition's cost model (PCG_RS_MODEL = K1 ocean chunk, K1 shared per
# chunk, K2/K3 ocean chunk, per overflow round, K2/K3 shared per chunk; us) on cfg4 AINV:
# loop us per iteration of the second solve.
for m in "$@"; do
  r=$(PCG_RS_MODEL=$m timeout 60 python tools/rs_one.py cfg4 ainv 2>&1 | tail -1)
  echo "$m  $r"
done
