mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c1.csv python tools/profile_solve.py --config c1_poisson7_64 --graph 0 > gpurun_out/ncu_c1_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c1.csv 27 > gpurun_out/launches_c1_summary.txt
