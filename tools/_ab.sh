b() { timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/ab_$1.json 2>/dev/null; }
for i in 1 2; do
  PM2L_LIB_PATH=$PWD/paper_2603_00549_b200/libpm2l_prev.so b prev$i
  b cur$i
done
