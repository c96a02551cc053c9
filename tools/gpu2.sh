mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
for bt in 4 6 8 10; do timeout 300 python bench.py --steps 3 --warmup 3 --bt $bt --no-cpu-baseline --no-e2e >> gpurun_out/bench_bt.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --T 40 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:an5d_sweep2d -s 5 -c 1 -o gpurun_out/prof_star2d1r python bench.py --steps 1 --warmup 1 --T 40 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
