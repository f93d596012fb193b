#!/bin/bash
# Re-run every bench.py workload once (1 GPU) and keep the JSON lines under
# gpurun_out/final_<name>.json; copied to profiles/r01_bench_<name>.json here.
set -u
mkdir -p gpurun_out
run() { local name=$1; shift; timeout 900 python bench.py "$@" > "gpurun_out/final_$name.json" 2> "gpurun_out/final_$name.err"; echo "$name rc=$?"; }
run mm
run tf32 --workload mm --precision tf32
run exact --workload mm --precision exact
run conv_bf16 --workload conv
run conv --workload conv --precision exact
run ls --workload ls
run linear32 --workload linear32
run ewise --workload ewise
run sweep --workload sweep
run reference_mm --impl reference
