#!/bin/bash
# Same-box comparison of several libcsa builds on the bench layer: scripts/ab_multi.sh LIB... ;
# each LIB is a path or "cur" (the tree's build).  Extra env for every run: $RUN_ENV.
for i in 1 2; do
  for L in "$@"; do
    if [ "$L" = cur ]; then P=""; else P=$PWD/$L; fi
    echo -n "$L: "; env $RUN_ENV CSA_LIB=$P ORDER=2 MODES=0 timeout 100 python scripts/pipe_bench.py
  done
done
