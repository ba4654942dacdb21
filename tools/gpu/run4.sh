mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fullsize_parity.py -m gpu -x -q -k "c1_poisson7_64 or c2_hetero27_128" > gpurun_out/gputest_full_c12.log 2>&1
tail -5 gpurun_out/gputest_full_c12.log
timeout 900 python bench.py --config c2_hetero27_128 --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -3 gpurun_out/bench_c2.err
python tools/layouts.py c2_hetero27_128 --time > gpurun_out/layouts_c2.json 2>&1
