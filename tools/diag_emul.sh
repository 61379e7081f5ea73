mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_reference_suites.py -q -m gpu -p no:cacheprovider > gpurun_out/refsuites.log 2>&1; tail -5 gpurun_out/refsuites.log
oracle/_ref/test_bandit_b200 2>&1 | tail -5
NCU=/usr/local/cuda/bin/ncu
for n in 1 2; do
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/emu${n}_launches.csv \
   python bench.py --emulate-world $n --weak --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-check --eager > gpurun_out/emu${n}_ncu.log 2>&1
done
