lscpu > gpurun_out/box_lscpu.txt 2>&1
nproc >> gpurun_out/box_lscpu.txt
free -g >> gpurun_out/box_lscpu.txt
python -c "
import threadpoolctl, scipy.linalg, numpy
import json
print(json.dumps(threadpoolctl.threadpool_info()))
" > gpurun_out/box_blas.txt 2>&1
OPENBLAS_CORETYPE=SkylakeX python -c "
import threadpoolctl, scipy.linalg, numpy
import json
print(json.dumps(threadpoolctl.threadpool_info()))
" >> gpurun_out/box_blas.txt 2>&1
nvidia-smi >> gpurun_out/box_lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02a.log 2>&1
tail -3 gpurun_out/gputest_r02a.log
