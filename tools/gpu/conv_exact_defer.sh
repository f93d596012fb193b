# A/B against ab/libold.so, a build of the previous source made for the measurement
# (git stash; build; cp paper_2307_16080_b200/libb200k.so ab/libold.so); ab/ is not tracked.
for i in 1 2; do
echo "new:"; python tools/probe_conv_exact.py 256 0
echo "old:"; B200_LIB=$PWD/ab/libold.so python tools/probe_conv_exact.py 256 0
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "conv" > gpurun_out/ce_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/ce_tests.log
