#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "calibration" > gpurun_out/pytest_calib.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_calib.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/bench_quick.log 2>&1
timeout 900 python scripts/calib_bench.py --heads-per-rank 5 --json-out gpurun_out/calib_m5_rank5.json > gpurun_out/calib_m5_rank5.log 2>&1
timeout 1500 python scripts/calib_bench.py --json-out gpurun_out/calib_m5_full.json > gpurun_out/calib_m5_full.log 2>&1
tail -n 3 gpurun_out/pytest_calib.log; tail -n 1 gpurun_out/bench_quick.log | cut -c1-300; tail -n 2 gpurun_out/calib_m5_rank5.log; tail -n 2 gpurun_out/calib_m5_full.log
