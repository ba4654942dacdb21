mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c3_ and not c4_" > gpurun_out/gputest_r02g.log 2>&1
tail -5 gpurun_out/gputest_r02g.log
python tools/layouts.py c2_hetero27_128 --time > gpurun_out/layouts_c2b.json 2>&1
python tools/layouts.py c2_hetero27_128 --time --opt wcsr=0 > gpurun_out/layouts_c2c.json 2>&1
python tools/tail_check.py c2_hetero27_128 "wcsr=0" "wcsr=1" > gpurun_out/wcsr_c2.txt 2>&1
