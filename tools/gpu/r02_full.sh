set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02b_gputests.log 2>&1; echo "pytest exit $?"
tail -8 gpurun_out/r02b_gputests.log
timeout 600 python tools/profile_sweep.py 48 > gpurun_out/r02_profile_sweep.txt 2>&1; echo "prof exit $?"
