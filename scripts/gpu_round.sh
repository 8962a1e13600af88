bash scripts/gpu_check.sh
bash scripts/gpu_bench.sh r01i wan720
for c in wan480 mochi; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --json-out gpurun_out/bench_r01i_$c.json > gpurun_out/bench_r01i_$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_r01i.log 2>&1
