# A/B the replay step over library variants: bash tools/ab.sh [variant ...]
# (variant = suffix of paper_2604_08706_b200/libreplay_b200_<v>.so, "cur" = the
# in-tree library, "cur:ENV=1" = the in-tree library with an env switch)
run() { timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1000,2), 'loss', round(d['roofline']['kernel_ms']*1000,2))"; }
vs=${@:-old cur}
for i in 1 2 3; do
  for v in $vs; do
    case $v in
      cur) run cur ;;
      cur:*) env ${v#cur:} bash -c "$(declare -f run); run $v" ;;
      *) REPLAY_B200_LIB=$PWD/paper_2604_08706_b200/libreplay_b200_$v.so run $v ;;
    esac
  done
done
