timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/full_gputests.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/full_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "smoke exit $?"
