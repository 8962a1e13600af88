#!/bin/bash
# Bench (all legs) + launch list + one full ncu capture of the attention and calibration kernels.
# Usage: gpu_bench.sh TAG [config]
TAG=${1:-r01}; CFG=${2:-wan720}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
timeout 900 python bench.py --config $CFG --steps 10 --warmup 3 --json-out gpurun_out/bench_${TAG}_${CFG}.json > gpurun_out/bench_${TAG}_${CFG}.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_${TAG}_${CFG}.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv python bench.py --config $CFG --steps 3 --warmup 1 --no-extras > gpurun_out/launches_${TAG}_${CFG}.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/launches_${TAG}_${CFG}.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-sparse_attn_sepp} -s 1 -c 1 -o gpurun_out/prof_attn_${TAG}_${CFG} -f python bench.py --config $CFG --steps 1 --warmup 1 --no-extras > gpurun_out/prof_attn_${TAG}_${CFG}.log 2>&1
echo "ncu full exit $?" >> gpurun_out/prof_attn_${TAG}_${CFG}.log
tail -n 3 gpurun_out/bench_${TAG}_${CFG}.log
