# A/B against ab/libold.so, a build of the previous source made for the measurement
# (git stash; build; cp paper_2307_16080_b200/libb200k.so ab/libold.so); ab/ is not tracked.
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullsize.py tests/test_gpu_tiled.py -x -q -p no:cacheprovider > gpurun_out/sh_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/sh_tests.log
for i in 1 2; do for lib in new old; do
if [ $lib = old ]; then export B200_LIB=$PWD/ab/libold.so; else unset B200_LIB; fi
timeout 300 python bench.py --workload ls --precision bf16 --min-seconds 1.0 > gpurun_out/sh.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/sh.json').read().strip().splitlines()[-1]); print('$lib', round(d['value']/1e3,1), d['roofline']['frac'], d['step_kernels_ms'], d['clocks']['sm_mhz'])"
done; done
