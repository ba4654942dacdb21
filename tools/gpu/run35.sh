# final validation: full GPU suite, bench lines (both arms) of the headline, bench lines of configs 1-3
mkdir -p gpurun_out
( time timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r02_final.log 2>&1 ) 2> gpurun_out/gputest_time.txt
echo "rc=$?" >> gpurun_out/gputest_r02_final.log
tail -4 gpurun_out/gputest_r02_final.log; cat gpurun_out/gputest_time.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
( time python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4_final.json 2> gpurun_out/bench_c4_final.err ) 2> gpurun_out/bench_time.txt
tail -c 400 gpurun_out/bench_c4_final.json; cat gpurun_out/bench_time.txt
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_c4_ref_final.json 2> gpurun_out/bench_c4_ref_final.err
for c in c2_hetero27_128 c1_poisson7_64 c3_elasticity_64; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_${c}_final.json 2> gpurun_out/bench_${c}_final.err
done
