mkdir -p gpurun_out
for v in d86 d66 d85; do
AMGB200_LIB=paper_2102_07417_b200/libamgb200_$v.so python tools/layouts.py t_rtanis7_256x64 --time > gpurun_out/layouts_$v.json 2>&1
done
python tools/layouts.py t_rtanis7_256x64 --time > gpurun_out/layouts_d55.json 2>&1
AMGB200_LIB=paper_2102_07417_b200/libamgb200_d86.so python tools/tail_check.py c4_rtanis7_256 "dict=1" > gpurun_out/c4_d86.txt 2>&1
cat gpurun_out/c4_d86.txt
python tools/tail_check.py c4_rtanis7_256 "dict=1" > gpurun_out/c4_d55.txt 2>&1
cat gpurun_out/c4_d55.txt
