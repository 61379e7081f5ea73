for n in 1 2 4 8; do
  timeout 400 python bench.py --emulate-world $n --steps 20 --no-e2e --no-cpu-baseline 2>gpurun_out/emu_$n.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($n, round(d['ms_per_step']*1000,2), '%.3g'%d['value'], d['config']['workload'][:40])" || tail -3 gpurun_out/emu_$n.err
done
RB_BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e > gpurun_out/same2.json 2> gpurun_out/same2.err; tail -c 600 gpurun_out/same2.json; tail -3 gpurun_out/same2.err
