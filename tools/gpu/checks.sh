# the parity suite against the AMG_CHECKS build (device-side invariant checks; compute-sanitizer is closed on this pool)
mkdir -p gpurun_out
AMGB200_LIB=paper_2102_07417_b200/libamgb200_checks.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not c4_" > gpurun_out/gputest_checks.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_checks.log
tail -5 gpurun_out/gputest_checks.log
