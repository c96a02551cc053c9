#!/bin/bash
# One parametrised gpurun session (run from the repo root on the GPU box):
#   bash tools/gpu_check.sh TAG MODE [MODE ...]
# MODES (run in the order given; outputs under gpurun_out/TAG_*):
#   tests      all -m gpu tests                     newrows  tests of the round-2 rows only
#   smoke      __graft_entry__.smoke()              bench    default bench line (+ e2e, cpu_baseline)
#   reference  bench --impl reference (CPU oracle)  ncu      ncu launch list of the default bench +
#                                                            ncu --set full of NCU_CASE (sweeponly.py args)
#   suite      bench --suite "$SUITE" (default all,config4) one line per workload
#   fmaform    FMA-pipe operand-form microbenchmark (tools/fmaform.cu)
#   ab         A/B: bench $AB_ARGS with the default lib and with AN5D_LIB=$AB_LIB, $AB_REPS times
#   absuite    A/B: bench --suite $SUITE with the default lib and with AN5D_LIB=$AB_LIB, $AB_REPS times
#   abenv      A/B: bench $AB_ARGS with and without the environment setting $AB_ENV (e.g. AN5D_PDL=0)
#   graph      CUDA-graph bit-identity tests + bench with and without --graph, $AB_REPS times
#   probe      tools/xpair_probe.py (each 3D x-pair case in its own process)
TAG=${1:-run}; shift
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests)
      timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
      echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt ;;
    newrows)
      timeout 1200 python -m pytest tests -m gpu -q -k "system or cluster or gradient2d or set_comm" \
          > gpurun_out/${TAG}_pytest_newrows.txt 2>&1
      echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_newrows.txt ;;
    smoke)
      python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
      echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt ;;
    bench)
      python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.jsonl 2>> gpurun_out/${TAG}_bench.err ;;
    reference)
      python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/${TAG}_reference.jsonl 2>> gpurun_out/${TAG}_bench.err ;;
    ncu)
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
          python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_bench.log 2>&1
      ncu --set full --clock-control none --import-source on -k regex:an5d_sweep -s 4 -c 1 -o gpurun_out/${TAG}_prof \
          python tools/sweeponly.py ${NCU_CASE:-star2d1r f32 8 60 8 6 32} > gpurun_out/${TAG}_ncu_full.log 2>&1 ;;
    suite)
      python bench.py --suite ${SUITE:-all,config4} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
          > gpurun_out/${TAG}_suite.jsonl 2>> gpurun_out/${TAG}_suite.err ;;
    fmaform)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fmaform tools/fmaform.cu && /tmp/fmaform > gpurun_out/${TAG}_fmaform.jsonl 2>&1 ;;
    ab)
      for rep in $(seq ${AB_REPS:-2}); do
        python bench.py --no-cpu-baseline --no-e2e ${AB_ARGS} >> gpurun_out/${TAG}_ab_default.jsonl 2>> gpurun_out/${TAG}_ab.err
        AN5D_LIB=$PWD/${AB_LIB} python bench.py --no-cpu-baseline --no-e2e ${AB_ARGS} >> gpurun_out/${TAG}_ab_variant.jsonl 2>> gpurun_out/${TAG}_ab.err
      done ;;
    absuite)
      for rep in $(seq ${AB_REPS:-2}); do
        python bench.py --suite ${SUITE:-all} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_suite_default.jsonl 2>> gpurun_out/${TAG}_ab.err
        AN5D_LIB=$PWD/${AB_LIB} python bench.py --suite ${SUITE:-all} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_suite_variant.jsonl 2>> gpurun_out/${TAG}_ab.err
      done ;;
    abenv)
      for rep in $(seq ${AB_REPS:-3}); do
        python bench.py --no-cpu-baseline --no-e2e ${AB_ARGS} >> gpurun_out/${TAG}_ab_default.jsonl 2>> gpurun_out/${TAG}_ab.err
        env ${AB_ENV} python bench.py --no-cpu-baseline --no-e2e ${AB_ARGS} >> gpurun_out/${TAG}_ab_variant.jsonl 2>> gpurun_out/${TAG}_ab.err
      done ;;
    graph)
      python -m pytest tests -m gpu -q -k cuda_graph > gpurun_out/${TAG}_pytest_graph.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_graph.txt
      for rep in $(seq ${AB_REPS:-2}); do
        python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tune --bt 8 --h 45 --graph >> gpurun_out/${TAG}_ab_graph.jsonl 2>> gpurun_out/${TAG}_ab.err
        python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tune --bt 8 --h 45 >> gpurun_out/${TAG}_ab_stream.jsonl 2>> gpurun_out/${TAG}_ab.err
      done ;;
    probe)
      python tools/xpair_probe.py > gpurun_out/${TAG}_probe.txt 2>&1 ;;
  esac
done
