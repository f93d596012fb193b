timeout 900 python -m pytest tests/test_gpu_stream.py -x -q -p no:cacheprovider > gpurun_out/ks_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/ks_tests.log
for sh in ${SHAPES:-"4,2,3,1" "4,2,3,2" "4,2,3,4" "4,2,4,2"}; do
B200_STREAM_2D_SHAPE=$sh timeout 300 python bench.py --workload mm --precision exact --min-seconds 1.0 > gpurun_out/ks.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/ks.json').read().strip().splitlines()[-1]); print('$sh', d['e2e']['value'], d['e2e']['ms_per_step'])"
done
