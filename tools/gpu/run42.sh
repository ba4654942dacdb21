mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_device_parity.py tests/test_fullsize_parity.py -m gpu -x -q -p no:cacheprovider -k "uniform_sell or interior_boundary or (fullsize_spmv and (c2_ or c1_ or c3_)) or smoother or golden" > gpurun_out/c16_tests.log 2>&1
tail -3 gpurun_out/c16_tests.log
python tools/spmv_one.py c2_hetero27_128 0 g --opt sellu_c16=0 > gpurun_out/c16_time.txt 2>&1
python tools/spmv_one.py c2_hetero27_128 0 g --opt sellu_c16=1 >> gpurun_out/c16_time.txt 2>&1
cat gpurun_out/c16_time.txt
python tools/tail_check.py c4_rtanis7_256 "sellu_c16=0" "sellu_c16=1" > gpurun_out/c4_c16.txt 2>&1
cat gpurun_out/c4_c16.txt
python tools/tail_check.py c2_hetero27_128 "sellu_c16=0" "sellu_c16=1" > gpurun_out/c2_c16.txt 2>&1
cat gpurun_out/c2_c16.txt
