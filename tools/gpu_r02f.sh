#!/bin/bash
# gpurun session: new-row parity tests (systems, clusters, gradient2d, set_comm), cluster A/B
# bench lines after the split-phase barrier, FMA operand-form microbenchmark.
TAG=${1:-r02f}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "system or cluster or gradient2d or set_comm" > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fmaform tools/fmaform.cu && /tmp/fmaform > gpurun_out/${TAG}_fmaform.jsonl 2>&1
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
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
