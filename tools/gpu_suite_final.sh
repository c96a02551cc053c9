#!/bin/bash
# round-2 final suite at BASELINE sizes (T = 1000, tuned planner): every Table-2 stencil fp32/fp64,
# config 4 (partial sums on/off), gradient2d, multi-field systems
TAG=${1:-r02l}
mkdir -p gpurun_out
python bench.py --suite all,config4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_suite.jsonl 2> gpurun_out/${TAG}_suite.err
python bench.py --suite star2d1r-x2-f32-16384,box2d1r-x2-f32-16384,star2d1r-x2-f64-16384,box2d1r-x2-f64-16384 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_suite_systems.jsonl 2>> gpurun_out/${TAG}_suite.err
