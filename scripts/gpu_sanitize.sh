#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K="attention_tiny or repetitive_block128 or (rect_attention_against_oracle and (80 or 192)) or edge_layouts"
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/synccheck.log 2>&1
echo "synccheck exit $?" >> gpurun_out/synccheck.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "attention_tiny or repetitive_block128 or running_max_jumps" > gpurun_out/memcheck_attn5.log 2>&1
echo "memcheck attn5 exit $?" >> gpurun_out/memcheck_attn5.log
tail -n 4 gpurun_out/synccheck.log gpurun_out/memcheck_attn5.log
