#!/bin/bash
# A/B: pair items (attn6.cu, order 3) vs single items (attn5.cu, order 2) + pair parity tests;
# TRACE=1 adds the attn6 trace build timeline at the end.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "${PYK:-pair_items or (full_size and wan720) or structured}" > gpurun_out/pytest_pair.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_pair.log
tail -3 gpurun_out/pytest_pair.log
for rep in 1 2; do
for o in ${ORDERS:-2 3}; do
CSA_ORDER=$o timeout 300 python bench.py --config ${CFG:-wan720} --steps 10 --warmup 3 --no-extras > gpurun_out/ab_o${o}_$rep.log 2>&1
python -c "import json,sys; l=[x for x in open('gpurun_out/ab_o${o}_$rep.log') if x.startswith('{')]; d=json.loads(l[-1]); print('order $o', d['value'], d['ms_per_step'], d['clocks'], d.get('parity',{}).get('pass'))" 2>&1 | tail -1
done
done
if [ -n "$TRACE" ]; then
CSA_TRACE_BUILD=1 python -m paper_2603_05503_b200._build --force > /dev/null 2>&1
timeout 300 python scripts/trace_attn6.py ${CFG:-wan720} > gpurun_out/trace6.log 2>&1; cat gpurun_out/trace6.log
fi
