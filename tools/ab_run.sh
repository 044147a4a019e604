python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
b() { python bench.py --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value']/1e9, d['e2e']['value']/1e9, d['e2e']['ms_per_step'], d['e2e']['pageable']['ms_per_step'])"; }
for i in 1 2 3; do
PM2L_LIB_PATH=$PWD/paper_2603_00549_b200/libpm2l_prev.so b prev
b cur
done
