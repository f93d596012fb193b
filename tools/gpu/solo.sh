timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tiled or tc or fullsize or random" > gpurun_out/solo_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/solo_tests.log
for v in "B200_TC_SOLO_OFF=1" "B200_TC_SOLO=1"; do
env $v timeout 300 python bench.py --workload mm --tiles 4x16 --precision bf16 --min-seconds 0.5 > gpurun_out/solo.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/solo.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['roofline']['frac'], d['step_kernels_ms'], d.get('accuracy',{}).get('max_norm_err'), d['config']['plan'])"
done
