python -m pytest tests -m gpu -x -q 2>&1 | tail -1
b() { python bench.py --steps 50 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value']/1e9, d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3)"; }
for i in 1 2 3; do
PM2L_LIB_PATH=$PWD/paper_2603_00549_b200/libpm2l_prev.so b prev
b cur
done
