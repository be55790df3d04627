#!/bin/bash
# Phase split of pass 2 for probe builds x {plain, TMA loads}:  VARIANTS="p2t p2t_p6" tools/ph_sweep.sh [config]
c=${1:-c5}
for v in $VARIANTS; do
  for tio in 0 1; do
    echo "== $v tio=$tio"
    PASD_P2_TIO=$tio PASD_B200_LIB=$PWD/build/$v.so timeout 200 python tools/p2_phases.py $c 2>&1
  done
done
