python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do
for v in prev cur; do
 if [ $v = prev ]; then export PM2L_LIB_PATH=$PWD/paper_2603_00549_b200/libpm2l_prev.so; else unset PM2L_LIB_PATH; fi
 echo "$v $(python tools/bench_modes.py 2>&1 | grep 'C3 cut' | cut -c60-120)"
 python tools/c5.py 2>&1 | grep "cutlass_att\|C5 rank" | cut -c1-130
done; done
unset PM2L_LIB_PATH
python bench.py --steps 50 --warmup 5 2>&1 | tail -1 | cut -c1-250
