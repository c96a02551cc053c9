#!/bin/bash
# One gpurun session: GPU tests, smoke, default bench, ncu launch list + ncu --set full of the
# headline sweep.  usage (under gpurun): bash tools/gpu_check.sh TAG [tests] [bench] [ncu]
TAG=${1:-run}; shift
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests)
      python -m pytest tests -m gpu -q --durations=25 > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
      echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
      python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
      echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt ;;
    bench)
      python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
      python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/${TAG}_reference.jsonl 2>> gpurun_out/${TAG}_bench.err ;;
    ncu)
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
          python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_bench.log 2>&1
      ncu --set full --clock-control none --import-source on -k regex:an5d_sweep -s 4 -c 1 -o gpurun_out/${TAG}_prof \
          python tools/sweeponly.py ${NCU_CASE:-star2d1r f32 7 45 8 6} > gpurun_out/${TAG}_ncu_full.log 2>&1 ;;
  esac
done
# extra modes (run after the fixed ones): TAG suite3d / suite2d -> default-planner suite lines
for what in "$@"; do
  case $what in
    suite3d)
      python bench.py --suite all3d --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_suite3d.jsonl 2>> gpurun_out/${TAG}_suite.err
      python bench.py --suite all3d --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --nthr 256 > gpurun_out/${TAG}_suite3d_n256.jsonl 2>> gpurun_out/${TAG}_suite.err
      python bench.py --suite all3d --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --nthr 512 > gpurun_out/${TAG}_suite3d_n512.jsonl 2>> gpurun_out/${TAG}_suite.err ;;
    suite2d)
      python bench.py --suite all2d,config4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_suite2d.jsonl 2>> gpurun_out/${TAG}_suite.err ;;
  esac
done
for what in "$@"; do
  case $what in
    split2d)
      for w in star2d1r-f32-16384 star2d1r-f64-16384 star2d2r-f32-16384 star2d2r-f64-16384 box2d1r-f32-16384 j2d5pt-f32-16384 j2d9pt-f32-16384; do
        for n in 32 64; do
          python bench.py --workload $w --nthr $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_split2d.jsonl 2>> gpurun_out/${TAG}_suite.err
        done
      done ;;
  esac
done
for what in "$@"; do
  case $what in
    boxhi)
      for w in box3d2r-f32-512 box3d3r-f32-512 box3d4r-f32-512 box3d3r-f64-512 box3d4r-f64-512; do
        python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_boxhi.jsonl 2>> gpurun_out/${TAG}_suite.err
      done ;;
  esac
done
for what in "$@"; do
  case $what in
    split1)
      for n in 32 64; do
        python bench.py --workload star2d1r-f32-16384 --nthr $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_split1.jsonl 2>> gpurun_out/${TAG}_suite.err
        python bench.py --workload star2d1r-f32-16384 --nthr $n --bt 7 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_split1.jsonl 2>> gpurun_out/${TAG}_suite.err
      done
      for w in j3d27pt-f64-512 box3d1r-f64-512 star3d3r-f64-512 box3d4r-f32-512 box3d4r-f64-512 box3d3r-f32-512; do
        python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_split1.jsonl 2>> gpurun_out/${TAG}_suite.err
      done ;;
  esac
done
for what in "$@"; do
  case $what in
    ab2d)
      for rep in 1 2; do
        python bench.py --workload star2d1r-f32-16384 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_ab2d.jsonl 2>> gpurun_out/${TAG}_suite.err
        AN5D_LIB=$PWD/paper_2001_01473_b200/libAN5D_noswap.so python bench.py --workload star2d1r-f32-16384 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_ab2d_noswap.jsonl 2>> gpurun_out/${TAG}_suite.err
      done
      for w in box3d1r-f64-512 j3d27pt-f64-512 star3d1r-f64-512 star2d2r-f32-16384 box2d1r-f32-16384; do
        python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_ab2d.jsonl 2>> gpurun_out/${TAG}_suite.err
      done ;;
  esac
done
for what in "$@"; do
  case $what in
    suiteall)
      python bench.py --suite all,config4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_suite.jsonl 2>> gpurun_out/${TAG}_suite.err ;;
    swapab)
      for rep in 1 2 3; do
        python bench.py --bt 7 --h 45 --nthr 32 --no-tune --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_swapab.jsonl 2>> gpurun_out/${TAG}_suite.err
        AN5D_LIB=$PWD/paper_2001_01473_b200/libAN5D_noswap.so python bench.py --bt 7 --h 45 --nthr 32 --no-tune --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_swapab_noswap.jsonl 2>> gpurun_out/${TAG}_suite.err
      done ;;
    ncufinal)
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
          python bench.py --bt 7 --h 45 --nthr 32 --no-tune --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_bench.log 2>&1
      ncu --set full --clock-control none --import-source on -k regex:an5d_sweep -s 4 -c 1 -o gpurun_out/${TAG}_prof_headline \
          python tools/sweeponly.py star2d1r f32 7 45 8 6 32 > gpurun_out/${TAG}_ncu_full.log 2>&1 ;;
  esac
done
for what in "$@"; do
  case $what in
    peerab)
      for rep in 1 2 3; do
        python bench.py --bt 7 --h 45 --nthr 32 --no-tune --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_peerab.jsonl 2>> gpurun_out/${TAG}_suite.err
        AN5D_LIB=$PWD/paper_2001_01473_b200/libAN5D_nopeer.so python bench.py --bt 7 --h 45 --nthr 32 --no-tune --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_peerab_nopeer.jsonl 2>> gpurun_out/${TAG}_suite.err
      done
      for rep in 1 2; do
        python bench.py --workload box3d2r-f64-512 --bt 1 --h 96 --nthr 256 --no-tune --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_peerab.jsonl 2>> gpurun_out/${TAG}_suite.err
        AN5D_LIB=$PWD/paper_2001_01473_b200/libAN5D_nopeer.so python bench.py --workload box3d2r-f64-512 --bt 1 --h 96 --nthr 256 --no-tune --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_peerab_nopeer.jsonl 2>> gpurun_out/${TAG}_suite.err
      done
      for w in j2d5pt-f32-16384 star2d3r-f32-16384 j2d9pt-f32-16384 star2d1r-f64-16384; do
        AN5D_TUNE_LOG=1 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_tune.jsonl 2>> gpurun_out/${TAG}_tune.err
      done ;;
  esac
done
