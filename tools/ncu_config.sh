# Full ncu captures of chosen kernels under one bench config (1 GPU).
#   CFG=c3 KERNELS="k_loss_grpo_buf k_gather" bash tools/ncu_config.sh
out=gpurun_out; mkdir -p $out
NCU=/usr/local/cuda/bin/ncu
for k in $KERNELS; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"$k" -s ${SKIP:-4} -c 1 \
      -o $out/prof_${CFG}_$k -f python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-check --eager \
      > $out/ncu_${CFG}_$k.log 2>&1
  echo "$CFG $k: $(ls -la $out/prof_${CFG}_$k.ncu-rep 2>/dev/null | awk '{print $5}')"
done
