timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02f_gputests.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r02f_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke exit $?"
timeout 1200 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference > gpurun_out/r02f_bench_ref.json 2> gpurun_out/r02f_bench_ref.err; echo "ref exit $?"; tail -c 600 gpurun_out/r02f_bench_ref.json
