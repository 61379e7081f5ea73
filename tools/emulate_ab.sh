# Emulated rank-0 step time for N GPUs under env variants:
#   bash tools/emulate_ab.sh "2 4 8" "" "RB_NO_LOOKAHEAD=1"
ns=$1; shift
for v in "$@"; do
  for n in $ns; do
    env $v timeout 400 python bench.py --emulate-world $n --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N=$n', '[$v]', round(d['ms_per_step']*1000,2))"
  done
done
