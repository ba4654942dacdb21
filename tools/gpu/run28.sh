mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "sorted_sell_in_steps" > gpurun_out/sellr_tests.log 2>&1
tail -8 gpurun_out/sellr_tests.log
for r in 2 3 4; do
python tools/layouts.py t_rtanis7_256x64 c2_hetero27_128 --time --opt sellr=$r --opt sells_max_rows=100000000 --opt sells_sigma=32 --opt sells_max_pad=100000 > gpurun_out/layouts_sellr$r.json 2>&1
done
python tools/layouts.py t_rtanis7_256x64 c2_hetero27_128 --time --opt sellr=3 > gpurun_out/layouts_sellr3_default.json 2>&1
