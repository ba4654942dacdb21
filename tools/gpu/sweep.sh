# usage: bash tools/gpu/sweep.sh CONFIG "opt1 opt2" "opt1 opt2" ...   (each arg = one option set)
cfg=$1; shift
mkdir -p gpurun_out
for set in "$@"; do
  args=""
  for o in $set; do args="$args --opt $o"; done
  v=$(timeout 600 python bench.py --config $cfg --steps 5 --warmup 2 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],4), d['iterations'])")
  echo "$cfg [$set] $v" >> gpurun_out/sweep.txt
done
