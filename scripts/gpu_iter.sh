#!/bin/bash
# Fast iteration: build, GPU tests, one bench line (no extras), optional ncu capture of attention.
TAG=${1:-iter}; CFG=${2:-wan720}; NCU=${3:-0}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
tail -n 4 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-extras > gpurun_out/bench_${TAG}_${CFG}.log 2>&1
tail -n 2 gpurun_out/bench_${TAG}_${CFG}.log
if [ "$NCU" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-sparse_attn_fixed_ref} -s 1 -c 1 -o gpurun_out/prof_attn_${TAG}_${CFG} -f python bench.py --config $CFG --steps 1 --warmup 1 --no-extras > gpurun_out/prof_attn_${TAG}_${CFG}.log 2>&1
echo "ncu exit $?"
fi
