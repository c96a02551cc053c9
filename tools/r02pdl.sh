# round 2 (r02pdl): programmatic dependent launch between sweeps -- GPU tests, then the default
# bench with PDL on / off interleaved (3 x), and a few suite rows both ways
bash tools/gpu_check.sh r02pdl tests
for rep in 1 2 3; do
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/r02pdl_ab_on.jsonl 2>> gpurun_out/r02pdl_ab.err
  AN5D_PDL=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/r02pdl_ab_off.jsonl 2>> gpurun_out/r02pdl_ab.err
done
S=star3d1r-f32-512,box3d1r-f32-512,star2d1r-f64-16384,star3d4r-f32-512
python bench.py --suite $S --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/r02pdl_suite_on.jsonl 2>> gpurun_out/r02pdl_ab.err
AN5D_PDL=0 python bench.py --suite $S --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/r02pdl_suite_off.jsonl 2>> gpurun_out/r02pdl_ab.err
