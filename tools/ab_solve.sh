# same-box A/B of whole-solve device time: bash tools/ab_solve.sh CONFIG "opt1" "opt2" ...
cfg=$1; shift
for rep in 1 2; do for o in "$@"; do
  printf "%-40s " "$o"; python tools/profile_solve.py --config $cfg --graph 2 --solves 3 $( [ -n "$o" ] && for kv in $o; do printf -- "--opt %s " $kv; done ) 2>&1 | tail -1 | cut -c1-48
done; done
