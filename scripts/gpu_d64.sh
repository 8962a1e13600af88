#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rect or denoise" > gpurun_out/pytest_d64.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_d64.log
timeout 300 python scripts/block_sweep.py --bkv 128,64,192 --d 64 > gpurun_out/d64_rect.log 2>&1
tail -n 2 gpurun_out/smoke.log; tail -n 3 gpurun_out/pytest_d64.log; cat gpurun_out/d64_rect.log | cut -c1-330
