mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "dict or class or golden" > gpurun_out/dict_tests.log 2>&1
tail -2 gpurun_out/dict_tests.log
for c in 0 1; do
python tools/layouts.py t_rtanis7_256x64 --time --opt dict_pf=$c > gpurun_out/layouts_dictpf$c.json 2>&1
done
python tools/tail_check.py c4_rtanis7_256 "dict_pf=0" "dict_pf=1" > gpurun_out/c4_pf.txt 2>&1
cat gpurun_out/c4_pf.txt
