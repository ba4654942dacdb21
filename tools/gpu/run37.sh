mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py tests/test_fullsize_parity.py -m gpu -x -q -p no:cacheprovider -k "sym or stencil or c2_ or hetero" > gpurun_out/symd27_tests.log 2>&1
tail -3 gpurun_out/symd27_tests.log
python tools/spmv_one.py c2_hetero27_128 0 a --opt symd_fast=0 > gpurun_out/symd27_time.txt 2>&1
python tools/spmv_one.py c2_hetero27_128 0 a --opt symd_fast=1 >> gpurun_out/symd27_time.txt 2>&1
cat gpurun_out/symd27_time.txt
python tools/tail_check.py c2_hetero27_128 "symd_fast=0" "symd_fast=1" > gpurun_out/symd27_c2.txt 2>&1
cat gpurun_out/symd27_c2.txt
