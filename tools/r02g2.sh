# round 2 (r02graph): CUDA-graph capture of the T-step run -- bit-identity tests, smoke, and the
# default bench with and without --graph, interleaved
python -m pytest tests -m gpu -q -k "cuda_graph or xpair" > gpurun_out/r02graph_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02graph_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02graph_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r02graph_smoke.txt
for rep in 1 2; do
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tune --bt 8 --h 45 --graph >> gpurun_out/r02graph_ab_graph.jsonl 2>> gpurun_out/r02graph_ab.err
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tune --bt 8 --h 45 >> gpurun_out/r02graph_ab_stream.jsonl 2>> gpurun_out/r02graph_ab.err
done
