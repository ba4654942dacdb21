mkdir -p gpurun_out
for o in coarse_pipe=1 coarse_pipe=0 coarse_pipe=20 coarse_pipe=100 tail_prefetch=0; do
AMGB200_TRACE=1 python tools/trace_tail.py c2_hetero27_128 $o 2>&1 | tail -2 | head -1 | sed "s/^/$o /" | grep -o "^[^ ]* .*coarse0/188:[0-9.]*us" | sed 's/spmv.*coarse/coarse/' >> gpurun_out/trace_coarse.txt
done
python tools/time_coarse.py c2_hetero27_128 >> gpurun_out/trace_coarse.txt 2>&1
