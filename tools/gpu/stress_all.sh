# Every randomized stress tool with fresh seeds, plus the extended random-shape
# suite; summary lines only (profiles/r02_stress.txt holds one run's output).
timeout 600 python tools/stress_sweep.py 400 101 2>&1 | tail -1
timeout 600 python tools/stress_plancache.py 1500 77 2>&1 | tail -1
timeout 600 python tools/stress_exact_tiles.py 150 55 2>&1 | tail -1
timeout 600 python tools/stress_conv_fused.py 200 66 2>&1 | tail -1
timeout 900 python tools/stress_shard.py 60 88 2>&1 | tail -1
timeout 600 python tools/stress_stream.py 300 99 2>&1 | tail -1
timeout 600 python tools/stress_races.py 300 12 2>&1 | tail -1
timeout 600 python tools/stress_tc.py 300 21 2>&1 | tail -1
B200_RANDOM_SCALE=50 B200_RANDOM_OFFSET=100000 timeout 2000 python -m pytest tests/test_gpu_random_shapes.py -q -p no:cacheprovider 2>&1 | tail -1
