timeout 900 python -m pytest tests/test_gpu_sweep.py -q -p no:cacheprovider > gpurun_out/sweep_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/sweep_tests.log
python bench.py --workload sweep > gpurun_out/sweep_n1.json 2>gpurun_out/sweep_n1.err; echo "exit $?"
python -c "
import json; d=json.loads(open('gpurun_out/sweep_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['phases_s_max_rank'], d['rank0_per_target_s'])"
