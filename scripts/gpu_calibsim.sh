#!/bin/bash
# Fused calibration + similarity: parity tests and timing against the two calls.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "${PYK:-calib_sim or calibration or similarity}" > gpurun_out/pytest_cs.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_cs.log; tail -15 gpurun_out/pytest_cs.log
timeout 300 python scripts/calib_time.py ${CFG:-wan720} > gpurun_out/cs_time.log 2>&1; cat gpurun_out/cs_time.log
