#!/bin/bash
# full GPU suite + default bench + 2D suite after the uniform-register change
TAG=${1:-r02g}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
python bench.py --suite all2d --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_suite2d.jsonl 2>> gpurun_out/${TAG}_bench.err
