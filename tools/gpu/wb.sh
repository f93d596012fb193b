timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_shard.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/wb_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/wb_tests.log
for w in ${WL:-"ls bf16" "ls exact" "mm exact" "conv bf16"}; do set -- $w
timeout 300 python bench.py --workload $1 --precision $2 --min-seconds 1.0 > gpurun_out/wb.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/wb.json').read().strip().splitlines()[-1]); print('$w', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],3))"
done
