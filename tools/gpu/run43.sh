mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 1500 --csv --log-file gpurun_out/launches_c4_final.csv python tools/profile_solve.py --config c4_rtanis7_256 --graph 0 > gpurun_out/ncu_c4_launch_final.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c4_final.csv > gpurun_out/launches_c4_final_summary.txt 2>&1
head -28 gpurun_out/launches_c4_final_summary.txt
cap() {
  ncu --set full --import-source on --clock-control none -k regex:$2 -s 3 -c 1 -o /tmp/$1 -f python tools/spmv_one.py c4_rtanis7_256 $3 $4 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>&1
  rm -f /tmp/$1.ncu-rep
}
cap c4_g1_sellu spmv_sellu 1 g
cap c4_p0_sellu_vd spmv_sellu 0 p
