#!/bin/bash
# Same-box comparison of calibration-pass builds at Wan 720p: scripts/ab_calib.sh LIB... ("cur"
# = the tree's build).
for i in 1 2; do
  for L in "$@"; do
    if [ "$L" = cur ]; then P=""; else P=$PWD/$L; fi
    echo -n "$L: "; CSA_LIB=$P timeout 100 python scripts/calib_run.py wan720 3 single | tail -1
  done
done
