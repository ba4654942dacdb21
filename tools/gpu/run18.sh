mkdir -p gpurun_out
python tools/layouts.py t_rtanis7_256x64 --time > gpurun_out/layouts_t4.json 2> gpurun_out/layouts_t4.err
python bench.py --config t_rtanis7_256x64 --steps 5 --warmup 3 > gpurun_out/bench_t4.json 2> gpurun_out/bench_t4.err
tail -c 1500 gpurun_out/bench_t4.json
python tools/profile_solve.py --help > gpurun_out/profile_help.txt 2>&1
