mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "uniform_sell or interior_boundary or golden or vcycle or smoother" > gpurun_out/vd_tests.log 2>&1
tail -4 gpurun_out/vd_tests.log
python tools/layouts.py c4_rtanis7_256 --time > gpurun_out/layouts_c4_vd.json 2> gpurun_out/layouts_c4_vd.err
python tools/tail_check.py c4_rtanis7_256 "sellu_vdict=0" "sellu_vdict=1" > gpurun_out/c4_vd.txt 2>&1
cat gpurun_out/c4_vd.txt
