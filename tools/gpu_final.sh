#!/bin/bash
# Round-2 final evidence on one B200: GPU tests, smoke, default bench (+ e2e, cpu_baseline),
# reference arm, ncu launch list of the default bench, ncu --set full of the headline sweep.
TAG=${1:-r02final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/${TAG}_reference.jsonl 2>> gpurun_out/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:an5d_sweep -s 4 -c 1 -o gpurun_out/${TAG}_prof_headline \
    python tools/sweeponly.py ${NCU_CASE:-star2d1r f32 8 60 8 6 32} > gpurun_out/${TAG}_ncu_full.log 2>&1
