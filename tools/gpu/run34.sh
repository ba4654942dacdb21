mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "dict or class or golden or smoother or hierarchy" > gpurun_out/dict_tests.log 2>&1
tail -3 gpurun_out/dict_tests.log
for c in 0 1; do
python tools/layouts.py t_rtanis7_256x64 c1_poisson7_64 --time --opt dict_shfl=$c > gpurun_out/layouts_dictsh$c.json 2>&1
done
python tools/tail_check.py c4_rtanis7_256 "dict_shfl=0" "dict_shfl=1" > gpurun_out/c4_shfl.txt 2>&1
cat gpurun_out/c4_shfl.txt
