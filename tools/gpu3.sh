mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 1200 python bench.py --suite all --steps 2 --warmup 1 > gpurun_out/suite.log 2>&1
ls -la gpurun_out
