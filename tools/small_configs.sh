# Per-config step / phase times and ncu launch lists for C1, C2, C3 (1 GPU).
#   bash tools/small_configs.sh [configs...]
out=gpurun_out; mkdir -p $out
NCU=/usr/local/cuda/bin/ncu
for c in ${@:-c1 c2 c3}; do
  for ph in "" "--phases"; do
    timeout 300 python bench.py --config $c --steps 50 --no-e2e --no-cpu-baseline --no-check $ph 2>$out/sc_$c.err | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({'config': '$c', 'phases': bool('$ph'), 'us_per_step': round(d['ms_per_step'] * 1e3, 2),
  'phases_us': {k: round(v * 1e3, 2) for k, v in d['phases_ms'].items() if isinstance(v, float)},
  'loss_kernel_us': round(d['roofline']['kernel_ms'] * 1e3, 2), 'step_frac': round(d['roofline']['step']['frac'], 3)}))" || tail -3 $out/sc_$c.err
  done
  timeout 300 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:'^(rb::)?k_|k_' -c 120 --csv --log-file $out/sc_${c}_launches.csv \
     python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-check --eager > $out/sc_${c}_ncu.log 2>&1
done
