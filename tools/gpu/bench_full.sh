nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python bench.py > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err; echo "bench exit $?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke2.log 2>&1; echo "smoke exit $?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv --log-file gpurun_out/r02_launches_default.csv python bench.py > gpurun_out/r02_ncu_default.log 2>&1; echo "ncu exit $?"
