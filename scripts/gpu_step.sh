#!/bin/bash
# f4 round trip: build, dictionary/denoise-step GPU test, step benchmark.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "denoise" > gpurun_out/pytest_step.log 2>&1
echo "pytest step exit $?" >> gpurun_out/pytest_step.log
timeout 1200 python scripts/step_bench.py --json-out gpurun_out/step_bench.json > gpurun_out/step_bench.log 2>&1
echo "step bench exit $?" >> gpurun_out/step_bench.log
tail -n 15 gpurun_out/pytest_step.log; tail -n 8 gpurun_out/step_bench.log
