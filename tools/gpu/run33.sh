# config 4: launch list + ncu full captures, exported as text on the box (reports are ~30 MB each)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "uniform_sell or sorted_sell" > gpurun_out/sellu_tests2.log 2>&1
tail -2 gpurun_out/sellu_tests2.log
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 2200 --csv --log-file gpurun_out/launches_c4.csv python tools/profile_solve.py --config c4_rtanis7_256 --graph 0 > gpurun_out/ncu_c4_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c4.csv > gpurun_out/launches_c4_summary.txt 2>&1
cap() {  # name regex level slot
  ncu --set full --import-source on --clock-control none -k regex:$2 -s 3 -c 1 -o /tmp/$1 -f python tools/spmv_one.py c4_rtanis7_256 $3 $4 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>&1
  rm -f /tmp/$1.ncu-rep
}
cap c4_a1_wcsr spmv_wcsr 1 a
cap c4_a0_dict spmv_dict 0 a
cap c4_p0_sellu spmv_sellu 0 p
ls -la gpurun_out | tail -12
