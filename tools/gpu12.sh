# source-level ncu capture of the default 2D sweep (per-instruction stall attribution)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:an5d_sweep -s 2 -c 1 -o gpurun_out/prof12_star2d1r python tools/cfgsweep.py star2d1r f32 7 8 128 0 2 > gpurun_out/ncu12.log 2>&1
ncu -i gpurun_out/prof12_star2d1r.ncu-rep --page source --csv --print-source sass > gpurun_out/prof12_sass.csv 2>&1
ls -la gpurun_out
