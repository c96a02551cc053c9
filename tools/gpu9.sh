# round check: parity, default bench, launch list, full ncu of the default sweep + star3d1r, suite
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi9.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu9.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu9.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench9.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches9.csv python bench.py --steps 1 --warmup 3 --T 40 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch9.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:an5d_sweep -s 2 -c 1 -o gpurun_out/prof9_star2d1r python tools/cfgsweep.py star2d1r f32 7 8 128 0 2 > gpurun_out/ncu9_2d.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:an5d_sweep -s 2 -c 1 -o gpurun_out/prof9_star3d1r python tools/cfgsweep.py star3d1r f32 3 2 64 0 2 > gpurun_out/ncu9_3d.log 2>&1
timeout 1800 python bench.py --suite all --steps 2 --warmup 1 > gpurun_out/suite9.log 2>&1
timeout 300 python bench.py --suite config4 --steps 2 --warmup 1 > gpurun_out/config4_9.log 2>&1
ls -la gpurun_out
