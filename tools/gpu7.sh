mkdir -p gpurun_out
timeout 300 python /root/repo/tools/dbg_direct.py > gpurun_out/dbg_direct.log 2>&1
(
timeout 600 python tools/cfgsweep.py star3d1r f32 3,4,5,6 2,4 64,128 0 5
timeout 300 python tools/cfgsweep.py star2d1r f32 4,5,6,7,8 4,8 0 0 5
) > gpurun_out/cfgsweep7.log 2>&1
timeout 1500 python bench.py --suite all --steps 2 --warmup 1 > gpurun_out/suite7.log 2>&1
ls -la gpurun_out
