set -x
timeout 900 python -m pytest tests/test_gpu_sweep.py -q -p no:cacheprovider > gpurun_out/sweep_tests.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/sweep_tests.log
B200_SWEEP_RESIDENT=0 python bench.py --workload sweep > gpurun_out/sweep_host.json 2>gpurun_out/sweep_host.err; echo "exit $?"
python bench.py --workload sweep > gpurun_out/sweep_res.json 2>gpurun_out/sweep_res.err; echo "exit $?"
python - <<'PY'
import json
for f in ("gpurun_out/sweep_host.json","gpurun_out/sweep_res.json"):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["phases_s_max_rank"], d["trials_only_configs_per_s"])
PY
timeout 600 python tools/profile_sweep.py 48 > gpurun_out/r02_profile_sweep_res.txt 2>&1; echo "prof exit $?"
