set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "c1_poisson7_64 or not fullsize" > gpurun_out/gputest_r02b.log 2>&1
tail -5 gpurun_out/gputest_r02b.log
timeout 600 python bench.py --config c1_poisson7_64 --steps 10 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
tail -3 gpurun_out/bench_c1.err
timeout 600 python bench.py --config c1_poisson7_64 --impl reference --steps 5 --warmup 2 > gpurun_out/bench_c1_ref.json 2>&1
