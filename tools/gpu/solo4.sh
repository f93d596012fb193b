python tools/probe_gemm.py --kind 0 --variant 2 3 --init 0 1 > gpurun_out/solo4_probe.log 2>&1; cat gpurun_out/solo4_probe.log
python tools/probe_gemm.py --kind 1 --variant 2 3 --init 0 >> gpurun_out/solo4_probe.log 2>&1; tail -2 gpurun_out/solo4_probe.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tiled or tc" > gpurun_out/solo_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/solo_tests.log
timeout 300 python bench.py --workload mm --tiles 4x16 --precision bf16 --min-seconds 0.5 > gpurun_out/solo.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/solo.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['step_kernels_ms'], d.get('accuracy',{}).get('max_norm_err'), d['config']['plan'])"
