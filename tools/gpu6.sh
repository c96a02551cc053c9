# parity (incl. the direct-gather variant) + configuration exploration for 3D and box2d2r on/off
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu6.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu6.log
(
timeout 300 python tools/cfgsweep.py box2d2r f32 1,2,3,4 4,8 0 0,1 5
timeout 300 python tools/cfgsweep.py box2d2r f64 1,2,3 4 0 0,1 5
timeout 300 python tools/cfgsweep.py star2d3r f32 1,2,3 4,8 0 0 5
timeout 600 python tools/cfgsweep.py star3d1r f32 1,2,3,4,5,6 2,4 32,64,128 0 5
timeout 600 python tools/cfgsweep.py star3d1r f64 1,2,3,4 2 32,64,128 0 5
timeout 300 python tools/cfgsweep.py box3d1r f32 1,2,3,4 2,4 32,64 0 5
timeout 300 python tools/cfgsweep.py star3d2r f32 1,2,3,4 2,4 32,64 0 5
) > gpurun_out/cfgsweep6.log 2>&1
timeout 900 python bench.py --suite box2d2r-f32-16384,box2d3r-f32-16384,box2d4r-f32-16384,box2d3r-f64-16384,star2d3r-f32-16384,star2d2r-f64-16384 --steps 2 --warmup 1 > gpurun_out/suite6.log 2>&1
ls -la gpurun_out
