#!/bin/bash
# Calibration scratch in L2: parity tests, timing, DRAM bytes per launch of both kernels (ncu).
TAG=${1:-r02d}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "calib or similarity" > gpurun_out/pytest_cs.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_cs.log; tail -2 gpurun_out/pytest_cs.log
timeout 300 python scripts/calib_time.py wan720 wan480
for K in calib_kernel calib_sim_kernel; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:$K -c 1 python scripts/calib_once.py wan720 2>&1 | grep -E "dram__|gpu__time|lts__t_sector|cycles_elapsed" 
done
