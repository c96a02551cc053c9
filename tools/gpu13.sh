# run-schedule check: new parity test, then star2d1r/box2d1r sweeps with runs off / on
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "runs or write_count or star2d1r" > gpurun_out/pytest13.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest13.log
for f in 0 0.85 0.93; do
  echo "== frac $f" >> gpurun_out/exp13.log
  AN5D_RUN_FRAC=$f timeout 300 python tools/cfgsweep.py star2d1r f32 5,6,7,8 8 32,64,128 0 6 >> gpurun_out/exp13.log 2>&1
done
for f in 0 0.85; do
  echo "== box2d1r frac $f" >> gpurun_out/exp13.log
  AN5D_RUN_FRAC=$f timeout 300 python tools/cfgsweep.py box2d1r f32 3,4,5 8 32,64,128 0 6 >> gpurun_out/exp13.log 2>&1
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench13.log 2>&1
ls -la gpurun_out
