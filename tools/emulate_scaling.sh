# Emulated multi-GPU evidence: rank 0 of an N-GPU job alone on
# one GPU (no collective), N = 1, 2, 4, 8, strong scaling (BASELINE configs[3]:
# the 16384 buffer and B = 4096 split N ways) and weak scaling.  Each line
# carries the step time and the per-phase split (front end = insert + sample +
# gather; loss) from events inside the graph.
#   bash tools/emulate_scaling.sh > gpurun_out/scaling_emulated.jsonl
for mode in strong weak; do
  for n in 1 2 4 8; do
    extra=""; [[ $mode == weak ]] && extra="--weak"
    for ph in "" "--phases"; do
      timeout 400 python bench.py --emulate-world $n --steps 20 --no-e2e --no-cpu-baseline --no-check $extra $ph \
        2>gpurun_out/emu_${mode}_$n.err | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({'mode': '$mode', 'N': $n, 'phases': bool('$ph'), 'us_per_step': round(d['ms_per_step'] * 1e3, 2),
                  'tokens_per_s_job': d['value'], 'phases_us': {k: round(v * 1e3, 2) for k, v in d['phases_ms'].items() if isinstance(v, float)},
                  'workload': d['config']['workload']}))" || tail -3 gpurun_out/emu_${mode}_$n.err
    done
  done
done
