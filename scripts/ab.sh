#!/bin/bash
# A/B: current tree vs tmp_v3 (older kernel) on the same box, same config, back to back.
CFG=${1:-wan720}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
(cd tmp_v3 && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/build_v3.log 2>&1)
for i in 1 2; do
  echo "== current $CFG"; timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['clocks'])"
  echo "== v3 $CFG"; (cd tmp_v3 && timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['clocks'])")
done
