#!/bin/bash
# Round-end evidence: smoke, full GPU suite, bench lines (3 configs), reference arm, launch list,
# one ncu --set full capture of the production attention kernel.
TAG=${1:-r01k}
bash scripts/gpu_check.sh
cp gpurun_out/pytest_gpu.log gpurun_out/pytest_gpu_$TAG.log
bash scripts/gpu_bench.sh $TAG wan720
for c in wan480 mochi; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --json-out gpurun_out/bench_${TAG}_$c.json > gpurun_out/bench_${TAG}_$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_$TAG.log 2>&1
