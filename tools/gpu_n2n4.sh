#!/bin/bash
# gpurun session: N4 (multi-field systems) parity tests + bench lines, N2 cluster A/B bench lines.
TAG=${1:-n2n4}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "system or cluster or gradient2d" > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for w in star2d1r-x2-f32-16384 box2d1r-x2-f32-16384 star2d1r-x2-f64-16384 box2d1r-x2-f64-16384; do
  timeout 300 $B --workload $w >> gpurun_out/${TAG}_system.jsonl 2>> gpurun_out/${TAG}.err
done
for w in star3d1r-f32-512 star3d2r-f32-512 box3d1r-f32-512; do
  for bsy in 32 64 128; do
    timeout 300 $B --workload $w --bsy $bsy >> gpurun_out/${TAG}_cluster.jsonl 2>> gpurun_out/${TAG}.err
  done
done
for w in star3d1r-f64-512 star3d2r-f64-512 box3d1r-f64-512; do
  for bsy in 32 64; do
    timeout 300 $B --workload $w --bsy $bsy --nthr 512 >> gpurun_out/${TAG}_cluster.jsonl 2>> gpurun_out/${TAG}.err
  done
done
timeout 300 $B --workload star3d1r-f64-512 --bsy 64 --nthr 256 >> gpurun_out/${TAG}_cluster.jsonl 2>> gpurun_out/${TAG}.err
