# A/B over library variants / env switches for one config:
#   CFG=c3 bash tools/ab_cfg.sh cur "cur:RB_PAYLOAD_LSU=1" s4l2
run() { timeout 200 python bench.py --config ${CFG:-c4} --no-cpu-baseline --no-e2e --no-check --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1000,2), 'loss', round(d['roofline']['kernel_ms']*1000,2))"; }
for i in 1 2; do
  for v in "$@"; do
    case $v in
      cur) run cur ;;
      cur:*) env ${v#cur:} bash -c "CFG=$CFG; $(declare -f run); run '$v'" ;;
      *) REPLAY_B200_LIB=$PWD/paper_2604_08706_b200/libreplay_b200_$v.so run $v ;;
    esac
  done
done
