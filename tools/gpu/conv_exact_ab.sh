timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "conv" > gpurun_out/ce_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/ce_tests.log
for v in "B200_CONV_EXACT_TMA=0" "B200_CONV_EXACT_TMA=1"; do
env $v timeout 300 python bench.py --workload conv --precision exact --min-seconds 0.5 > gpurun_out/ce_$v.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/ce_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['roofline']['frac'], d['step_kernels_ms'], d.get('accuracy'))"
done
