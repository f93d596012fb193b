timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/e2e_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/e2e_tests.log
for v in "B200_STREAM_2D=0" "B200_STREAM_2D=1"; do
env $v timeout 600 python bench.py --workload mm --precision exact > gpurun_out/e2e_mm.json 2> gpurun_out/e2e_mm.err; echo "bench exit $?"
python -c "
import json; d=json.loads(open('gpurun_out/e2e_mm.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"
done
