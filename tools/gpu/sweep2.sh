set -x
python bench.py --workload sweep > gpurun_out/sweep_n1.json 2>gpurun_out/sweep_n1.err; echo "exit $?"
B200_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload sweep > gpurun_out/sweep_n2_gloo.json 2>gpurun_out/sweep_n2.err; echo "exit $?"
python - <<'PY'
import json
for f in ("gpurun_out/sweep_n1.json","gpurun_out/sweep_n2_gloo.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["phases_s_max_rank"], d["trials_only_configs_per_s"], d["config"]["parallelism"])
    except Exception as e: print(f, e)
PY
