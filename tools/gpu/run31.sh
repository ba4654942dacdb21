mkdir -p gpurun_out
python tools/layouts.py c4_rtanis7_256 --time --opt sells_max_rows=2000000 > gpurun_out/layouts_c4_sells2m.json 2> gpurun_out/layouts_c4_sells2m.err
python tools/tail_check.py c4_rtanis7_256 "sells_max_rows=2000000" "sells_max_rows=8000000" > gpurun_out/c4_sells.txt 2>&1
cat gpurun_out/c4_sells.txt
