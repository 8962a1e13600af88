python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in wan480 wan720; do for r in 4 0; do
timeout 300 python bench.py --config $c --rep-heads $r --no-extras --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c rep $r', d['value'], d['ms_per_step'], d['config']['kept_fraction'])"
done; done
