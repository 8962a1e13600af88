#!/bin/bash
# Same-box A/B of calibsim.cu variants (scripts/calib_time.py): the current build and variants
# built by scripts/build_variant.sh from $VARIANTS ("name|sed-expr;...") applied to calibsim.cu.
mkdir -p gpurun_out tmp_ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  n=${v%%|*}; e=${v#*|}
  bash scripts/build_variant.sh $n paper_2603_05503_b200/csrc/calibsim.cu "$e" > /dev/null 2>&1 || echo "build $n failed"
done
if [ -n "$PYK" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$PYK" > gpurun_out/pytest_cs.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_cs.log; tail -2 gpurun_out/pytest_cs.log
fi
for i in 1 2; do
  echo -n "main: "; timeout 200 python scripts/calib_time.py ${CFG:-wan720}
  for v in "${VS[@]}"; do n=${v%%|*}
    echo -n "$n: "; CSA_LIB=$PWD/tmp_ab/lib_$n.so timeout 200 python scripts/calib_time.py ${CFG:-wan720}
  done
done
