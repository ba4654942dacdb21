mkdir -p gpurun_out
python tools/spmv_one.py t_rtanis7_256x64 0 a > gpurun_out/spmv_one_t4_a0.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmv_dict -s 3 -c 1 -o gpurun_out/t4_a0_dict -f python tools/spmv_one.py t_rtanis7_256x64 0 a > gpurun_out/ncu_t4_a0.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmv_wcsr -s 3 -c 1 -o gpurun_out/t4_a1_wcsr -f python tools/spmv_one.py t_rtanis7_256x64 1 a > gpurun_out/ncu_t4_a1.log 2>&1
tail -3 gpurun_out/ncu_t4_a0.log
