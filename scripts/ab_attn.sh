#!/bin/bash
# Same-box A/B of the attention kernel: tmp_ab/libA.so (a reference build) vs the current
# libcsa.so, interleaved, on the bench config's layer (scripts/pipe_bench.py).  Extra env for
# the B side can be passed as $B_ENV (e.g. "CSA_EMU_EVERY=4").
for i in 1 2 3; do
  echo -n "A: "; CSA_LIB=$PWD/tmp_ab/libA.so ORDER=2 MODES=0 timeout 100 python scripts/pipe_bench.py
  echo -n "B: "; env $B_ENV ORDER=2 MODES=0 timeout 100 python scripts/pipe_bench.py
done
