# config 4 at full size: per-matrix timings, both bench arms, full-size parity, launch shares, ncu captures
mkdir -p gpurun_out
nproc > gpurun_out/c4_box.txt; free -g | head -2 >> gpurun_out/c4_box.txt
( time python tools/layouts.py c4_rtanis7_256 --time > gpurun_out/layouts_c4.json 2> gpurun_out/layouts_c4.err ) 2>> gpurun_out/c4_box.txt
( time python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err ) 2>> gpurun_out/c4_box.txt
tail -c 800 gpurun_out/bench_c4.json
( time python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_c4_ref.json 2> gpurun_out/bench_c4_ref.err ) 2>> gpurun_out/c4_box.txt
tail -c 600 gpurun_out/bench_c4_ref.json
( time timeout 2400 python -m pytest tests/test_fullsize_parity.py -m gpu -x -q -p no:cacheprovider -k c4 > gpurun_out/gputest_c4.log 2>&1 ) 2>> gpurun_out/c4_box.txt
tail -5 gpurun_out/gputest_c4.log
cat gpurun_out/c4_box.txt
