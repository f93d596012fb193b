for v in "4,2,3" "8,2,4" "8,4,6" "4,4,4" "8,4,8" "16,4,8"; do
B200_STREAM_2D_SHAPE=$v timeout 600 python bench.py --workload mm --precision exact --steps 5 --min-seconds 0.5 > gpurun_out/e2e_mm.json 2> gpurun_out/e2e_mm.err
python -c "
import json; d=json.loads(open('gpurun_out/e2e_mm.json').read().strip().splitlines()[-1]); print('$v', d['e2e']['value'], d['e2e']['ms_per_step'])"
done
