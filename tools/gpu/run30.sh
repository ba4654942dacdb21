# config 4 profiles: eager launch list (natural cache state) + full captures of the top kernels
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 4000 --csv --log-file gpurun_out/launches_c4.csv python tools/profile_solve.py --config c4_rtanis7_256 --graph 0 > gpurun_out/ncu_c4_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c4.csv > gpurun_out/launches_c4_summary.txt 2>&1
head -30 gpurun_out/launches_c4_summary.txt
ncu --set full --import-source on --clock-control none -k regex:spmv_wcsr -s 3 -c 1 -o gpurun_out/c4_a1_wcsr -f python tools/spmv_one.py c4_rtanis7_256 1 a > gpurun_out/ncu_c4_a1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmv_dict -s 3 -c 1 -o gpurun_out/c4_a0_dict -f python tools/spmv_one.py c4_rtanis7_256 0 a > gpurun_out/ncu_c4_a0.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmv_sellu -s 3 -c 1 -o gpurun_out/c4_g1_sellu -f python tools/spmv_one.py c4_rtanis7_256 1 g > gpurun_out/ncu_c4_g1.log 2>&1
ls -la gpurun_out/*.ncu-rep
