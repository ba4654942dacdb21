mkdir -p gpurun_out
AMGB200_DEBUG=1 timeout 1200 python -m pytest tests -m gpu -x -q -s -k "nccl_calls" > gpurun_out/gputest_r02e.log 2>&1
tail -15 gpurun_out/gputest_r02e.log
timeout 600 python bench.py --config c2_hetero27_128 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2b.json 2> gpurun_out/bench_c2b.err
tail -3 gpurun_out/bench_c2b.err
