mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "jds or interior_boundary_split_spmv" > gpurun_out/jds_tests.log 2>&1
tail -5 gpurun_out/jds_tests.log
for mb in 2 3 4; do
python tools/layouts.py c2_hetero27_128 c3_elasticity_64 c1_poisson7_64 --time --opt jds=3 --opt jds_minb=$mb > gpurun_out/layouts_jds3_mb$mb.json 2>&1
done
python tools/tail_check.py c2_hetero27_128 "jds=1" "jds=3" "jds=1 jds_minb=2" > gpurun_out/jds_c2.txt 2>&1
cat gpurun_out/jds_c2.txt
python tools/tail_check.py c3_elasticity_64 "jds=1" "jds=3" > gpurun_out/jds_c3.txt 2>&1
cat gpurun_out/jds_c3.txt
