#!/bin/bash
# ncu evidence after the uniform-register change + the 3D suite:
#   launch list of the default bench, ncu --set full of the headline sweep (NCU_CASE = "name dt bT h vec n nthr"),
#   3D suite at the planner's pick, ncu --set full of the 3D fp64 star sweeps and box3d4r fp32.
TAG=${1:-r02h}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "edge_cases or decoupled or set_comm" > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:an5d_sweep -s 4 -c 1 -o gpurun_out/${TAG}_prof_headline \
    python tools/sweeponly.py ${NCU_CASE:-star2d1r f32 7 45 8 6 32} > gpurun_out/${TAG}_ncu_full.log 2>&1
python bench.py --suite all3d --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_suite3d.jsonl 2>> gpurun_out/${TAG}.err
ncu --set full --clock-control none --import-source on -k regex:an5d_sweep -s 4 -c 1 -o gpurun_out/${TAG}_prof_s3d2r_f64 \
    python tools/sweeponly.py star3d2r f64 2 64 2 6 512 > gpurun_out/${TAG}_ncu_s3d2r.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:an5d_sweep -s 4 -c 1 -o gpurun_out/${TAG}_prof_s3d1r_f64 \
    python tools/sweeponly.py star3d1r f64 3 64 2 6 512 > gpurun_out/${TAG}_ncu_s3d1r.log 2>&1
python bench.py --suite config4,gradient2d-f32-16384,gradient2d-f64-16384,star2d1r-x2-f32-16384,box2d1r-x2-f32-16384,star2d1r-x2-f64-16384,box2d1r-x2-f64-16384 \
    --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_suite_extra.jsonl 2>> gpurun_out/${TAG}.err
