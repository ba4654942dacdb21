mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c3_ and not c4_" > gpurun_out/gputest_r02f.log 2>&1
tail -5 gpurun_out/gputest_r02f.log
