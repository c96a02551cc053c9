# final check of the committed library: parity suite, smoke, default bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu21.log 2>&1
echo pytest rc=$? >> gpurun_out/pytest_gpu21.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke21.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench21.log 2>&1
timeout 300 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/ref21.log 2>&1
ls -la gpurun_out
