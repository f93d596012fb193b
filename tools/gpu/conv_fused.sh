set -x
timeout 300 python -m pytest tests/test_gpu_conv.py -x -q -p no:cacheprovider -k "bf16 or tc" > gpurun_out/cf_tests.log 2>&1; echo "conv tests exit $?"; tail -5 gpurun_out/cf_tests.log
timeout 300 python bench.py --workload conv --precision bf16 > gpurun_out/cf_bench_fused.json 2> gpurun_out/cf_bench_fused.err; echo "fused bench exit $?"
B200_CONV_UNFUSED=1 timeout 300 python bench.py --workload conv --precision bf16 > gpurun_out/cf_bench_unfused.json 2> gpurun_out/cf_bench_unfused.err; echo "unfused bench exit $?"
python - <<'PY'
import json
for f in ("gpurun_out/cf_bench_fused.json","gpurun_out/cf_bench_unfused.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"]/1e3,1), "TF", d["ms_per_step"], d["step_kernels_ms"], d["roofline"]["frac"], d.get("accuracy"), d["config"]["plan"])
    except Exception as e: print(f, e)
PY
