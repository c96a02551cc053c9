# register-budget / level-skew experiment on star2d1r fp32 (exp libraries from AN5D_BUILD_TAG builds)
mkdir -p gpurun_out
for lib in "" f12 sk f12sk; do
  if [ -z "$lib" ]; then L=paper_2001_01473_b200/libAN5D.so; else L=paper_2001_01473_b200/libAN5D_$lib.so; fi
  echo "== lib ${lib:-base}" >> gpurun_out/exp11.log
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py star2d1r f32 3,4,5,6,7,8 8 128,256 0 6 >> gpurun_out/exp11.log 2>&1
done
ls -la gpurun_out
