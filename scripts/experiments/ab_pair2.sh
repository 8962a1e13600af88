#!/bin/bash
# Same-box A/B of attn6 variants (pipe_bench.py, Wan 720p layer): attn5 (order 2), attn6 (order 3)
# and variants built by scripts/build_variant.sh from $VARIANTS ("name|sed-expr;name|sed-expr").
mkdir -p gpurun_out tmp_ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  n=${v%%|*}; e=${v#*|}
  bash scripts/build_variant.sh $n paper_2603_05503_b200/csrc/attn6.cu "$e" > /dev/null 2>&1 || echo "build $n failed"
done
if [ -n "$PYK" ]; then
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$PYK" > gpurun_out/pytest_pair.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_pair.log; tail -2 gpurun_out/pytest_pair.log
fi
for i in 1 2; do
  echo -n "attn5: "; ORDER=2 MODES=0 timeout 100 python scripts/pipe_bench.py ${CFG:-wan720}
  echo -n "attn6: "; ORDER=3 MODES=0 timeout 100 python scripts/pipe_bench.py ${CFG:-wan720}
  for v in "${VS[@]}"; do n=${v%%|*}
    echo -n "$n: "; CSA_LIB=$PWD/tmp_ab/lib_$n.so ORDER=3 MODES=0 timeout 100 python scripts/pipe_bench.py ${CFG:-wan720}
  done
done
if [ -n "$TRACE" ]; then
CSA_TRACE_BUILD=1 python -m paper_2603_05503_b200._build --force > /dev/null 2>&1
timeout 300 python scripts/trace_attn6.py ${CFG:-wan720} > gpurun_out/trace6.log 2>&1; cat gpurun_out/trace6.log
fi
