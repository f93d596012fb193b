for i in 1 2; do for gm in 8 16; do
B200_TC2_GROUP=$gm timeout 300 python bench.py --workload mm --precision bf16 --min-seconds 1.0 > gpurun_out/g.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('mm group $gm', round(d['value']/1e3,1), d['roofline']['frac'], d['step_kernels_ms'], d['clocks']['sm_mhz'])"
done; done
for gm in 8 16; do
B200_TC2_GROUP=$gm timeout 300 python bench.py --workload ls --precision bf16 --min-seconds 1.0 > gpurun_out/g.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('ls group $gm', round(d['value']/1e3,1), d['roofline']['frac'], d['step_kernels_ms'], d['clocks']['sm_mhz'])"
done
