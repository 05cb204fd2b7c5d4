#!/bin/bash
# ncu evidence for the hot-path kernels (run under gpurun, 1 GPU):
#   launches.csv         every launch of a short default bench with its device time
#                        (cold-cache, serialised: compare SHARES, not absolutes)
#   <name>.ncu-rep       one `--set full` capture of each top kernel
# Usage: tools/profile.sh [launches] [gemm] [fa] [fp8] [moe] [ln] [md] [bwd] [simp]
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
NCU="ncu --clock-control none"
for what in "$@"; do
  case $what in
    launches)
      timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
        --log-file "$OUT/launches.csv" python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu \
        > "$OUT/launches_bench.log" 2>&1 ;;
    gemm)
      timeout 900 $NCU --set full --import-source on --kernel-name-base demangled \
        -k regex:"gemm_wide_kernel|gemm_bf16_kernel.*SchedT<.int.1>" -s 3 -c 1 -o "$OUT/gemm" -f \
        python bench.py --workload gemm --no-secondary --steps 2 --warmup 3 --no-e2e --no-cpu \
        > "$OUT/gemm_ncu.log" 2>&1 ;;
    fa)
      timeout 900 $NCU --set full --import-source on -k regex:attention_fwd_kernel -s 3 -c 1 \
        -o "$OUT/fa" -f python bench.py --workload attention --steps 1 --warmup 3 --no-cpu \
        > "$OUT/fa_ncu.log" 2>&1 ;;
    fp8)
      timeout 900 $NCU --set full --import-source on -k regex:mxfp8_kernel -s 3 -c 1 \
        -o "$OUT/fp8" -f python bench.py --workload fp8 --steps 1 --warmup 3 --no-cpu \
        > "$OUT/fp8_ncu.log" 2>&1 ;;
    moe)
      timeout 900 $NCU --set full --import-source on --kernel-name-base demangled \
        -k regex:"GroupedSched|GroupedWideSched" -s 3 -c 1 -o "$OUT/moe" -f \
        python bench.py --workload moe --steps 1 --warmup 3 --no-cpu > "$OUT/moe_ncu.log" 2>&1 ;;
    ln)
      timeout 900 $NCU --set full --import-source on -k regex:layernorm_cluster -s 3 -c 1 \
        -o "$OUT/ln" -f python bench.py --workload layernorm --steps 2 --warmup 3 --no-cpu \
        > "$OUT/ln_ncu.log" 2>&1 ;;
    md)
      timeout 900 $NCU --set full --import-source on --kernel-name-base demangled \
        -k regex:GatherSched -s 3 -c 1 -o "$OUT/md" -f \
        python bench.py --workload multidevice --steps 2 --warmup 3 --no-cpu > "$OUT/md_ncu.log" 2>&1 ;;
    bwd)
      timeout 900 $NCU --set full --import-source on -k regex:attention_bwd_kernel -s 1 -c 1 \
        -o "$OUT/bwd" -f python bench.py --workload attention_bwd --steps 3 --warmup 3 --no-cpu \
        > "$OUT/bwd_ncu.log" 2>&1 ;;
    simp)
      timeout 900 $NCU --set full --import-source on -k regex:simplicial -s 1 -c 1 \
        -o "$OUT/simp" -f python bench.py --workload simplicial --steps 3 --warmup 3 --no-cpu \
        > "$OUT/simp_ncu.log" 2>&1 ;;
  esac
  echo "$what rc=$?"
done
