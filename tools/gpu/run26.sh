mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "dict or class or golden or smoother or hierarchy" > gpurun_out/dict_tests.log 2>&1
tail -3 gpurun_out/dict_tests.log
for r in 1 2; do
python tools/layouts.py t_rtanis7_256x64 c1_poisson7_64 --time --opt dict_rows=$r > gpurun_out/layouts_dictml_r$r.json 2>&1
done
python tools/layouts.py t_rtanis7_256x64 --time --opt dict_rows=2 --opt dict_chunk=1 > gpurun_out/layouts_dictml_r2c.json 2>&1
python tools/tail_check.py t_rtanis7_256x64 "dict_rows=1" "dict_rows=2" "dict_main=0" > gpurun_out/dict_t4.txt 2>&1
cat gpurun_out/dict_t4.txt
python tools/tail_check.py c1_poisson7_64 "dict_rows=1" "dict_rows=2" "dict_main=0" > gpurun_out/dict_c1.txt 2>&1
cat gpurun_out/dict_c1.txt
