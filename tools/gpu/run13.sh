# session-4 sanity: full GPU suite + bench lines of configs 1-3 on a fresh box
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r02h.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_r02h.log
tail -5 gpurun_out/gputest_r02h.log
for c in c2_hetero27_128 c1_poisson7_64 c3_elasticity_64; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -c 600 gpurun_out/bench_$c.json
done
python tools/layouts.py c2_hetero27_128 c1_poisson7_64 c3_elasticity_64 --time > gpurun_out/layouts_r02h.json 2>&1
