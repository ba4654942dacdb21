mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "warp_cooperative or interior_boundary_split_spmv" > gpurun_out/wcsr2_tests.log 2>&1
tail -5 gpurun_out/wcsr2_tests.log
python tools/layouts.py c2_hetero27_128 c3_elasticity_64 --time --opt wcsr=2 > gpurun_out/layouts_wcsr2.json 2>&1
python tools/layouts.py c3_elasticity_64 --time --opt wcsr=2 --opt sells=0 --opt sell=0 --opt long_avg=0 > gpurun_out/layouts_wcsr2_c3all.json 2>&1
python tools/layouts.py c3_elasticity_64 --time --opt wcsr=1 --opt sells=0 --opt sell=0 --opt long_avg=0 > gpurun_out/layouts_wcsr1_c3all.json 2>&1
python tools/tail_check.py c2_hetero27_128 "wcsr=1" "wcsr=2" > gpurun_out/wcsr2_c2.txt 2>&1
cat gpurun_out/wcsr2_c2.txt
