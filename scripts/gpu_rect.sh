#!/bin/bash
# f3 round trip: build, rect + plan + merge GPU tests, whole GPU suite, block-size sweep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rect or merge or plan_compile" > gpurun_out/pytest_rect.log 2>&1
echo "pytest rect exit $?" >> gpurun_out/pytest_rect.log
timeout 600 python scripts/block_sweep.py --json-out gpurun_out/block_sweep.json > gpurun_out/block_sweep.log 2>&1
echo "sweep exit $?" >> gpurun_out/block_sweep.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -n 4 gpurun_out/pytest_rect.log; tail -n 12 gpurun_out/block_sweep.log; tail -n 3 gpurun_out/pytest_gpu.log
