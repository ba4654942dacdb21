mkdir -p gpurun_out
AMGB200_TRACE=1 python tools/trace_tail.py c2_hetero27_128 > gpurun_out/trace_c2.txt 2>&1
AMGB200_TRACE=1 python tools/trace_tail.py c1_poisson7_64 > gpurun_out/trace_c1.txt 2>&1
for g in 2 1; do python bench.py --config c2_hetero27_128 --steps 5 --warmup 3 --no-cpu-baseline --opt graph=$g > gpurun_out/bench_c2_graph$g.json 2>/dev/null; done
