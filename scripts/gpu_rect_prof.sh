#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rect_attention_against_oracle or rect_attention_overflow or (calibration_against_oracle and 128-80) or denoise" > gpurun_out/memcheck_rect.log 2>&1
echo "memcheck exit $?" >> gpurun_out/memcheck_rect.log
for b in 64 192; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn_rect -s 3 -c 1 -o gpurun_out/prof_attn_r01j_rect$b -f python scripts/block_sweep.py --bkv $b --steps 1 --warmup 1 > gpurun_out/prof_rect$b.log 2>&1
done
tail -n 4 gpurun_out/memcheck_rect.log; ls gpurun_out/*.ncu-rep
