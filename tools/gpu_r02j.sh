#!/bin/bash
# after the 3D dead-warp skip and the one-period 2D loop: full GPU suite, 3D suite, default bench
TAG=${1:-r02j}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
python bench.py --suite all3d --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_suite3d.jsonl 2>> gpurun_out/${TAG}.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.jsonl 2>> gpurun_out/${TAG}.err
