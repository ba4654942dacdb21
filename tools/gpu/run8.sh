mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:tail_vcycle -c 1 -o gpurun_out/tail_c2 -f python tools/trace_tail.py c2_hetero27_128 > gpurun_out/ncu_tail.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:coarse_solve_k -c 1 -o gpurun_out/coarse_c2 -f python tools/time_coarse.py c2_hetero27_128 > gpurun_out/ncu_coarse.log 2>&1
ls -la gpurun_out/*.ncu-rep
