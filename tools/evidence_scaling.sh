# Evidence for DESIGN §6: emulated rank-0 step at N = 1, 2, 4, 8 and a
# one-step timeline at N = 1 and N = 8 (debug clocks library).
bash tools/emulate_ab.sh "1 2 4 8" ""
for n in 1 8; do
  echo "== timeline, emulated N=$n"
  EMU_WORLD=$n STEPS=1 GRAPH=1 timeout 300 python tools/timeline.py 2>&1 | grep -v "^local"
done
