ncu --set full --clock-control none --import-source on -k regex:grid_ -s 2 -c 1 -o gpurun_out/grid_final -f python tools/profile_grid.py 5 > gpurun_out/gncu.log 2>&1
tail -2 gpurun_out/gncu.log
