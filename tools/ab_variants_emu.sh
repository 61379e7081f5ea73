for i in 1 2; do
for v in cur u8 u12; do
  for n in 1 2; do
    if [ $v = cur ]; then L=""; else L="REPLAY_B200_LIB=$PWD/paper_2604_08706_b200/libreplay_b200_$v.so"; fi
    env $L timeout 300 python bench.py --emulate-world $n --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v N=$n', round(d['ms_per_step']*1000,2))"
  done
done
done
