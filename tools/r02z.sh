# round 2 (r02z4): x-pair 3D tiles with 16-byte-aligned TMA boxes -- per-case probe, GPU tests,
# then the affected 3D rows with the new library and the previous one (AN5D_LIB), interleaved
python tools/xpair_probe.py > gpurun_out/r02z4_probe.txt 2>&1
bash tools/gpu_check.sh r02z4 tests
S=box3d1r-f32-512,j3d27pt-f32-512,star3d1r-f32-512,star3d2r-f32-512,box3d2r-f32-512
for rep in 1 2; do
  python bench.py --suite $S --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/r02z4_suite3d_xpair.jsonl 2>> gpurun_out/r02z4_suite.err
  AN5D_LIB=$PWD/paper_2001_01473_b200/libAN5D_comb.so python bench.py --suite $S --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/r02z4_suite3d_prev.jsonl 2>> gpurun_out/r02z4_suite.err
done
