mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -x -q -p no:cacheprovider -k "jds" > gpurun_out/jds_tests3.log 2>&1
tail -3 gpurun_out/jds_tests3.log
for mb in 2 3; do
python tools/layouts.py c2_hetero27_128 --time --opt jds=3 --opt jds_minb=$mb > gpurun_out/layouts_jdsL_mb$mb.json 2>&1
done
python tools/layouts.py c2_hetero27_128 --time --opt jds=3 --opt jds_minb=2 --opt jds_step=16 > gpurun_out/layouts_jdsL_s16.json 2>&1
