mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "uniform_sell or interior_boundary or golden or smoother or vcycle" > gpurun_out/sellu_tests.log 2>&1
tail -3 gpurun_out/sellu_tests.log
python tools/layouts.py c4_rtanis7_256 --time > gpurun_out/layouts_c4_v2.json 2> gpurun_out/layouts_c4_v2.err
python tools/tail_check.py c4_rtanis7_256 "sellu_sort=0" "sellu_sort=1" > gpurun_out/c4_sellu.txt 2>&1
cat gpurun_out/c4_sellu.txt
python tools/tail_check.py c2_hetero27_128 "sellu_sort=0" "sellu_sort=1" > gpurun_out/c2_sellu.txt 2>&1
cat gpurun_out/c2_sellu.txt
python tools/tail_check.py c3_elasticity_64 "sellu_sort=0" "sellu_sort=1" > gpurun_out/c3_sellu.txt 2>&1
cat gpurun_out/c3_sellu.txt
