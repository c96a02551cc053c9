#!/bin/bash
# gpurun session for the round-2 N2 (3D cluster halo sharing) and N3 (gradient2d) rows:
# their parity tests, then A/B bench lines (one block vs clusters; gradient2d per dtype).
TAG=${1:-n2n3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "gradient2d or cluster or exports" > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for w in star3d1r-f32-512 star3d2r-f32-512 box3d1r-f32-512 j3d27pt-f32-512; do
  for bsy in 32 64 128; do
    timeout 300 $B --workload $w --bsy $bsy >> gpurun_out/${TAG}_cluster.jsonl 2>> gpurun_out/${TAG}.err
  done
done
for w in star3d1r-f64-512 star3d2r-f64-512 box3d1r-f64-512 j3d27pt-f64-512; do
  for nt in 256 512; do
    for bsy in 32 64; do
      timeout 300 $B --workload $w --bsy $bsy --nthr $nt >> gpurun_out/${TAG}_cluster.jsonl 2>> gpurun_out/${TAG}.err
    done
  done
done
for w in gradient2d-f32-16384 gradient2d-f64-16384; do
  timeout 300 $B --workload $w >> gpurun_out/${TAG}_grad.jsonl 2>> gpurun_out/${TAG}.err
done
