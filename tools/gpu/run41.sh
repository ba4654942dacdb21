mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "warp_cooperative or interior_boundary" > gpurun_out/wbig_tests.log 2>&1
tail -3 gpurun_out/wbig_tests.log
python tools/spmv_one.py c4_rtanis7_256 2 a --opt sells_max_rows=1048576 --opt wcsr_big=0 > gpurun_out/wbig_a2.txt 2>&1
python tools/spmv_one.py c4_rtanis7_256 2 a --opt sells_max_rows=1048576 --opt wcsr_big=1 >> gpurun_out/wbig_a2.txt 2>&1
python tools/spmv_one.py c4_rtanis7_256 2 a >> gpurun_out/wbig_a2.txt 2>&1
python tools/spmv_one.py c4_rtanis7_256 1 a --opt wcsr_big=1 >> gpurun_out/wbig_a2.txt 2>&1
cat gpurun_out/wbig_a2.txt
