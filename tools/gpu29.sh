# outer unroll 2 on fp64 star r1, fp32 box r1, fp32 star r2
mkdir -p gpurun_out
for lib in "" u2b; do
  if [ -z "$lib" ]; then L=paper_2001_01473_b200/libAN5D.so; else L=paper_2001_01473_b200/libAN5D_$lib.so; fi
  echo "== lib ${lib:-base}" >> gpurun_out/exp29.log
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py star2d1r f64 6,7,8 4 64 0 8 >> gpurun_out/exp29.log 2>&1
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py box2d1r f32 3,4,5 8 40 0 8 >> gpurun_out/exp29.log 2>&1
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py star2d2r f32 3,4,5 8 60 0 8 >> gpurun_out/exp29.log 2>&1
done
