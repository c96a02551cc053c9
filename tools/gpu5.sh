# round check: tests, default bench, suite, launch list, full ncu captures of the 2D default and star3d1r
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 1500 python bench.py --suite all --steps 2 --warmup 1 > gpurun_out/suite.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --T 40 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:an5d_sweep -s 2 -c 1 -o gpurun_out/prof_default python bench.py --steps 1 --warmup 1 --T 40 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:an5d_sweep -s 2 -c 1 -o gpurun_out/prof_star3d1r python bench.py --workload star3d1r-f32-512 --steps 1 --warmup 1 --T 30 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full3d.log 2>&1
ls -la gpurun_out
