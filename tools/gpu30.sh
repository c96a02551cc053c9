# run-fraction sweep for the default workload with the v9 library
mkdir -p gpurun_out
for f in 0.75 0.85 0.93; do
  echo "== frac $f" >> gpurun_out/exp30.log
  AN5D_RUN_FRAC=$f timeout 300 python tools/cfgsweep.py star2d1r f32 7,8 8 32,48,60,96 0 8 >> gpurun_out/exp30.log 2>&1
done
