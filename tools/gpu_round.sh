#!/usr/bin/env bash
# One GPU measurement round (run under gpurun): tests, smoke, bench, ncu.
#   bash tools/gpu_round.sh [tests|bench|ncu|all] [extra bench args...]
set -u
what=${1:-all}
shift || true
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $out/gpu.txt 2>&1

if [[ $what == tests || $what == all ]]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 --durations=8 > $out/pytest_gpu.log 2>&1
  tail -15 $out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
  tail -3 $out/smoke.log
fi

if [[ $what == bench || $what == all ]]; then
  timeout 900 python bench.py "$@" > $out/bench.json 2> $out/bench.err
  tail -c 4000 $out/bench.json; tail -5 $out/bench.err
fi

if [[ $what == ncu || $what == all ]]; then
  NCU=/usr/local/cuda/bin/ncu
  rm -f $out/prof_*.ncu-rep $out/ncu_*.log
  # launch list of one short bench run (cold-cache, serialised: compare shares)
  timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:'^k_' -c 400 --csv --log-file $out/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-check --eager > $out/ncu_bench.log 2>&1
  echo "launches: $(grep -c k_ $out/launches.csv)"
  # full captures of the heavy kernels in steady state
  for k in ${NCU_KERNELS:-k_loss_grpo_buf k_gather k_insert_payload_tma k_route_fifo k_sample_fused}; do
    timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"^$k\$" -s 4 -c 1 \
        -o $out/prof_$k -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check --eager \
        > $out/ncu_$k.log 2>&1
    echo "$k: $(ls -la $out/prof_$k.ncu-rep 2>/dev/null | awk '{print $5}')"
  done
fi
