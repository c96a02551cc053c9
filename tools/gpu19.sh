# 3D run schedule: full parity suite, then star3d1r / box3d1r / star3d2r sweeps with runs off / on
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu19.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu19.log
for f in 0 0.85; do
  echo "== frac $f" >> gpurun_out/exp19.log
  AN5D_RUN_FRAC=$f timeout 300 python tools/cfgsweep.py star3d1r f32 2,3,4 2,4 16,32,64 0 6 >> gpurun_out/exp19.log 2>&1
  AN5D_RUN_FRAC=$f timeout 300 python tools/cfgsweep.py star3d2r f32 1,2 2 16,32,64 0 6 >> gpurun_out/exp19.log 2>&1
  AN5D_RUN_FRAC=$f timeout 300 python tools/cfgsweep.py star3d1r f64 2,3 2 16,32,64 0 6 >> gpurun_out/exp19.log 2>&1
done
ls -la gpurun_out
