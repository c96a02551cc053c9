# restored-state check: parity suite, default bench, config-5 (1536^3) bench at N=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi10.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu10.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu10.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench10.log 2>&1
timeout 900 python bench.py --workload star3d2r-f32-1536 --steps 3 --warmup 3 > gpurun_out/bench10_c5.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke10.log 2>&1
ls -la gpurun_out
