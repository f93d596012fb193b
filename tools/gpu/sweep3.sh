python bench.py --workload sweep > gpurun_out/sweep_n1.json 2>gpurun_out/sweep_n1.err; echo "exit $?"
for n in 2 8; do
B200_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --workload sweep > gpurun_out/sweep_n${n}_gloo.json 2>gpurun_out/sweep_n$n.err; echo "exit $?"
done
nproc
python - <<'PY'
import json
for f in ("gpurun_out/sweep_n1.json","gpurun_out/sweep_n2_gloo.json","gpurun_out/sweep_n8_gloo.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"],1), d["phases_s_max_rank"], d["rank0_per_target_s"], d["config"]["parallelism"])
    except Exception as e: print(f, e)
PY
