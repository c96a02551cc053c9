# outer stream-loop unroll 2 experiment (fewer back-edge register moves)
mkdir -p gpurun_out
for lib in "" u2; do
  if [ -z "$lib" ]; then L=paper_2001_01473_b200/libAN5D.so; else L=paper_2001_01473_b200/libAN5D_$lib.so; fi
  echo "== lib ${lib:-base}" >> gpurun_out/exp27.log
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py star2d1r f32 4,5,6,7,8 8 32,60 0 8 >> gpurun_out/exp27.log 2>&1
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py star2d1r f32 4,5,6,7,8 8 32,60 0 8 >> gpurun_out/exp27.log 2>&1
done
