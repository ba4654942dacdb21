mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "dict or class or golden or smoother" > gpurun_out/dict_tests.log 2>&1
tail -3 gpurun_out/dict_tests.log
for c in 0 1; do for r in 1 2; do
python tools/layouts.py t_rtanis7_256x64 c1_poisson7_64 --time --opt dict_rows=$r --opt dict_chunked=$c > gpurun_out/layouts_dictc${c}_r$r.json 2>&1
done; done
python tools/tail_check.py t_rtanis7_256x64 "dict_chunked=0" "dict_chunked=1" "dict_chunked=1 dict_rows=1" > gpurun_out/dict_t4.txt 2>&1
cat gpurun_out/dict_t4.txt
