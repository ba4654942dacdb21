mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "jds or warp_cooperative or interior_boundary_split_spmv" > gpurun_out/jds_tests2.log 2>&1
tail -5 gpurun_out/jds_tests2.log
python tools/layouts.py c2_hetero27_128 c3_elasticity_64 --time --opt jds=3 --opt jds_minb=2 --opt jds_step=16 > gpurun_out/layouts_jds3_s16.json 2>&1
python tools/layouts.py c2_hetero27_128 c3_elasticity_64 --time --opt wcsr=2 > gpurun_out/layouts_wcsrpf.json 2>&1
python tools/layouts.py c3_elasticity_64 --time --opt wcsr=2 --opt sells=0 --opt sell=0 > gpurun_out/layouts_wcsrpf_c3all.json 2>&1
python tools/tail_check.py c2_hetero27_128 "wcsr=2" "jds=1 jds_minb=2 jds_step=16" > gpurun_out/pf_c2.txt 2>&1
cat gpurun_out/pf_c2.txt
