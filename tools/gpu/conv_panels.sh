for prec in exact bf16; do for p in 8 16 32; do
B200_CONV_PANELS=$p timeout 300 python bench.py --workload conv --precision $prec --min-seconds 1.0 > gpurun_out/cp.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/cp.json').read().strip().splitlines()[-1]); print('$prec panels $p', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],3))"
done; done
