mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "c1_poisson7_64 or not fullsize" > gpurun_out/gputest_r02c.log 2>&1
tail -5 gpurun_out/gputest_r02c.log
timeout 600 python bench.py --config c1_poisson7_64 --steps 10 --warmup 3 > gpurun_out/bench_c1b.json 2> gpurun_out/bench_c1b.err
tail -3 gpurun_out/bench_c1b.err
