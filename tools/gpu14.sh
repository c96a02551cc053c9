# round check after the run schedule: parity, default bench, launch list, full ncu of the default sweep, 2D suite
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi14.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu14.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu14.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench14.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches14.csv python bench.py --steps 1 --warmup 3 --T 40 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch14.log 2>&1
BT=$(python -c "import json;d=json.loads(open('gpurun_out/bench14.log').read().strip().split(chr(10))[-1]);c=d['config'];print(c['bT'],c['vec'],c['h'])")
set -- $BT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:an5d_sweep -s 2 -c 1 -o gpurun_out/prof14_star2d1r python tools/cfgsweep.py star2d1r f32 $1 $2 $3 0 2 > gpurun_out/ncu14_2d.log 2>&1
ncu -i gpurun_out/prof14_star2d1r.ncu-rep --page source --csv --print-source sass > gpurun_out/prof14_sass.csv 2>&1
timeout 1800 python bench.py --suite all2d,config4 --steps 2 --warmup 1 > gpurun_out/suite14.log 2>&1
ls -la gpurun_out
