mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r02i.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_r02i.log
tail -4 gpurun_out/gputest_r02i.log
python tools/layouts.py t_rtanis7_256x64 --time --opt sells_max_rows=100000000 > gpurun_out/layouts_t4_sells.json 2>&1
python tools/layouts.py t_rtanis7_256x64 --time --opt sells_max_rows=100000000 --opt sells_sigma=32 --opt sells_max_pad=300 > gpurun_out/layouts_t4_sells32.json 2>&1
python tools/layouts.py t_rtanis7_256x64 --time > gpurun_out/layouts_t4_b.json 2>&1
python tools/tail_check.py t_rtanis7_256x64 "sells_max_rows=100000000" > gpurun_out/sells_t4.txt 2>&1
cat gpurun_out/sells_t4.txt
