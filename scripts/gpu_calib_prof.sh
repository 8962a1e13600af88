#!/bin/bash
# Calibration kernels: parity tests, timing, and one ncu --set full capture of each.
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "calib or similarity" > gpurun_out/pytest_cs.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_cs.log; tail -2 gpurun_out/pytest_cs.log
timeout 300 python scripts/calib_time.py wan720 wan480
for K in calib_kernel calib_sim_kernel; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_${K}_$TAG -f python scripts/calib_once.py wan720 > gpurun_out/prof_${K}_$TAG.log 2>&1
echo "ncu $K exit $?"
done
