mkdir -p gpurun_out
for v in 3 5 6; do
AMGB200_LIB=paper_2102_07417_b200/libamgb200_s$v.so python tools/spmv_one.py c2_hetero27_128 0 a > gpurun_out/symd27_minb$v.txt 2>&1; cat gpurun_out/symd27_minb$v.txt
done
