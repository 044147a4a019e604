python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step']*1e3, d['roofline']['frac'], d['roofline']['traffic'], d['e2e']['value']/1e9, d['gpu_launches'], d['clocks']['reasons'])"
