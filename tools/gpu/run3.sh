mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "c1_poisson7_64 or not fullsize" > gpurun_out/gputest_r02d.log 2>&1
tail -5 gpurun_out/gputest_r02d.log
timeout 600 python bench.py --config c1_poisson7_64 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1c.json 2> gpurun_out/bench_c1c.err
tail -3 gpurun_out/bench_c1c.err
python tools/layouts.py c1_poisson7_64 --time > gpurun_out/layouts_c1.json 2>&1
