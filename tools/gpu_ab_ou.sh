#!/bin/bash
# A/B: two-period stream loop (default for fp32 star b_T >= 6) vs one period (libAN5D_ou1.so)
TAG=${1:-abou}
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-tune --h 45 --nthr 32 --vec 8"
for rep in 1 2; do
  for bt in 8 7; do
    $B --bt $bt >> gpurun_out/${TAG}_default.jsonl 2>> gpurun_out/${TAG}.err
    AN5D_LIB=$PWD/paper_2001_01473_b200/libAN5D_ou1.so $B --bt $bt >> gpurun_out/${TAG}_ou1.jsonl 2>> gpurun_out/${TAG}.err
  done
done
