python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step']*1e3, json.dumps(d['e2e']))"
PM2L_E2E_TRACE=1 python bench.py --steps 4 --warmup 3 2>&1 | grep "pm2l drain" | tail -3
