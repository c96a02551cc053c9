# round-end measurements: default bench, config 5, smoke, launch list, ncu of the 3D sweep, full suite
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi20.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench20.log 2>&1
timeout 900 python bench.py --workload star3d2r-f32-1536 --steps 3 --warmup 3 > gpurun_out/bench20_c5.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke20.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches20.csv python bench.py --steps 1 --warmup 3 --T 40 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch20.log 2>&1
timeout 1800 python bench.py --suite all,config4 --steps 2 --warmup 1 > gpurun_out/suite20.log 2>&1
CFG=$(python -c "
import json
for l in open('gpurun_out/suite20.log'):
    try: d=json.loads(l)
    except Exception: continue
    c=d.get('config',{})
    if c.get('workload')=='star3d1r-f32-512': print(c['bT'],c['vec'],c['h'])")
set -- $CFG
timeout 600 ncu --set full --import-source on --clock-control none -k regex:an5d_sweep -s 2 -c 1 -o gpurun_out/prof20_star3d1r python tools/cfgsweep.py star3d1r f32 $1 $2 $3 0 2 > gpurun_out/ncu20_3d.log 2>&1
ls -la gpurun_out
