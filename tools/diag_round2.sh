out=gpurun_out; mkdir -p $out
bash tools/small_configs.sh c1 c2 c3 > $out/small_configs.jsonl 2>&1
for n in 1 8; do
  echo "== timeline strong emulated N=$n" >> $out/timelines.txt
  EMU_WORLD=$n STEPS=1 GRAPH=1 timeout 300 python tools/timeline.py >> $out/timelines.txt 2>&1
done
for c in c1 c3; do
  echo "== timeline $c" >> $out/timelines.txt
  CFG=$c STEPS=1 GRAPH=1 timeout 300 python tools/timeline.py >> $out/timelines.txt 2>&1
done
