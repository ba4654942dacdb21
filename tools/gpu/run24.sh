mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_device_setup.py -m gpu -x -q -p no:cacheprovider > gpurun_out/setup_tests.log 2>&1
tail -15 gpurun_out/setup_tests.log
python - > gpurun_out/load_times.txt 2>&1 <<'PY'
import time, os
from paper_2102_07417_b200 import hiercache
for cfg in ["c2_hetero27_128", "t_rtanis7_256x64"]:
    d = os.path.join("hier_cache", cfg)
    if not os.path.exists(d): continue
    for dev in (None, 0):
        t = time.time(); h = hiercache.load_hierarchy(d, device=dev); print(cfg, "device" if dev is not None else "host", round(time.time() - t, 1), "s", flush=True)
print("cpus", os.cpu_count())
PY
cat gpurun_out/load_times.txt
