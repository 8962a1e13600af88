#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the fused calibration + similarity
# tests (calibsim.cu) and the intervals-only plan attention tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K="calib_sim_fused_against_oracle and (lay0 or lay1 or lay2 or lay3 or lay4)"
for tool in memcheck racecheck synccheck; do
timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/${tool}_calibsim.log 2>&1
echo "$tool exit $?" >> gpurun_out/${tool}_calibsim.log
tail -n 3 gpurun_out/${tool}_calibsim.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "intervals_only_plan_bitwise" > gpurun_out/memcheck_intervals.log 2>&1
echo "memcheck intervals exit $?" >> gpurun_out/memcheck_intervals.log
tail -n 3 gpurun_out/memcheck_intervals.log
