#!/bin/bash
# A/B: star2d1r fp32 one-warp tiles of 256 cells (vec 8) vs 128 cells (vec 4, more warps per SM)
TAG=${1:-abv4}
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  $B --vec 8 --bt 8 >> gpurun_out/${TAG}.jsonl 2>> gpurun_out/${TAG}.err
  for bt in 6 7 8; do
    AN5D_LIB=$PWD/paper_2001_01473_b200/libAN5D_v4.so $B --vec 4 --bt $bt >> gpurun_out/${TAG}.jsonl 2>> gpurun_out/${TAG}.err
  done
done
AN5D_LIB=$PWD/paper_2001_01473_b200/libAN5D_v4.so $B >> gpurun_out/${TAG}_tuned.jsonl 2>> gpurun_out/${TAG}.err
