mkdir -p gpurun_out
for c in 0 1; do
python tools/layouts.py t_rtanis7_256x64 c1_poisson7_64 --time --opt dict_chunk=$c > gpurun_out/layouts_dictml_c$c.json 2>&1
done
python tools/tail_check.py t_rtanis7_256x64 "dict_chunk=0" "dict_chunk=1" > gpurun_out/dict_t4.txt 2>&1
cat gpurun_out/dict_t4.txt
