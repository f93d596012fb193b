#!/bin/bash
# Plain bench run, then (only if it exited 0) one `ncu --set full` capture of
# the workload's dominant kernel.  Run on the B200 box through gpurun; the
# bench lines land in gpurun_out/bench_<name>.json, the reports in
# gpurun_out/ncu_<name>.ncu-rep (read here with tools/ncu_traffic.py).
set -u
mkdir -p gpurun_out
cap() {  # name, kernel regex, count, bench args...
  local name=$1 kre=$2 cnt=$3; shift 3
  timeout 600 python bench.py "$@" > "gpurun_out/bench_$name.json" 2> "gpurun_out/bench_$name.err"
  local rc=$?
  echo "$name bench rc=$rc"
  [ $rc -eq 0 ] || return
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -c "$cnt" \
    -f -o "gpurun_out/ncu_$name" python bench.py "$@" --steps 1 --warmup 3 \
    > "gpurun_out/ncu_$name.log" 2>&1
  echo "$name ncu rc=$?"
}
if [ $# -gt 0 ]; then cap "$@"; exit; fi
cap mm_gemm_exact contract_exact 1 --workload mm --precision exact
cap mm_gemm_tf32 gemm_tc2 1 --workload mm --precision tf32
cap conv_conv_exact conv_exact_kernel 1 --workload conv
cap ls_gemm_bf16 gemm_tc2 2 --workload ls
cap ewise_map_exact b200_map_jit 1 --workload ewise
