python -m pytest tests/test_gpu_random_tables.py -m gpu -x -q -k row_block 2>&1 | tail -2
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 30 --warmup 5 2>&1 | tail -1 | cut -c1-200
