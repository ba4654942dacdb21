mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_fullsize_parity.py -m gpu -x -q -k "c3_" > gpurun_out/gputest_full_c3.log 2>&1
tail -5 gpurun_out/gputest_full_c3.log
timeout 900 python bench.py --config c3_elasticity_64 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python tools/layouts.py c3_elasticity_64 --time > gpurun_out/layouts_c3.json 2>&1
