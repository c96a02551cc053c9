# parity, default bench, suite (tuned planner), config 4, TMA 3D profile
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu8.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu8.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench8.log 2>&1
timeout 300 python bench.py --suite config4 --steps 2 --warmup 1 > gpurun_out/config4_8.log 2>&1
timeout 1800 python bench.py --suite all --steps 2 --warmup 1 > gpurun_out/suite8.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:an5d_sweep -s 2 -c 1 -o gpurun_out/prof8_star3d1r python tools/cfgsweep.py star3d1r f32 3 4 64 0 2 > gpurun_out/ncu8_3d.log 2>&1
ls -la gpurun_out
