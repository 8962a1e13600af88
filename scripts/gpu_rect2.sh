#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "calibration" > gpurun_out/pytest_calib_rect.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_calib_rect.log
timeout 900 python scripts/block_sweep.py --calibrated --json-out gpurun_out/block_sweep_calibrated.json > gpurun_out/block_sweep_calibrated.log 2>&1
echo "sweep exit $?" >> gpurun_out/block_sweep_calibrated.log
tail -n 15 gpurun_out/pytest_calib_rect.log; tail -n 12 gpurun_out/block_sweep_calibrated.log
