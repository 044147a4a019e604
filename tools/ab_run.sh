python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do
echo "prev $(PM2L_LIB_PATH=$PWD/paper_2603_00549_b200/libpm2l_prev.so python tools/bench_modes.py 2>&1 | grep points | cut -c1-200)"
echo "cur $(python tools/bench_modes.py 2>&1 | grep points | cut -c1-200)"
done
python tools/c4.py 2>&1 | tail -1 | cut -c1-200
