# seam layout experiment (all taps FFMA2) vs the pair layout, 2D fp32
mkdir -p gpurun_out
for lib in "" seam; do
  if [ -z "$lib" ]; then L=paper_2001_01473_b200/libAN5D.so; else L=paper_2001_01473_b200/libAN5D_$lib.so; fi
  echo "== lib ${lib:-base}" >> gpurun_out/exp15.log
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py star2d1r f32 5,6,7,8 8 60 0 6 >> gpurun_out/exp15.log 2>&1
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py box2d1r f32 3,4,5 8 40 0 6 >> gpurun_out/exp15.log 2>&1
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py box2d2r f32 1,2,3 8 60 0 6 >> gpurun_out/exp15.log 2>&1
  AN5D_LIB=$L timeout 300 python tools/cfgsweep.py star2d2r f32 2,3,4 8 60 0 6 >> gpurun_out/exp15.log 2>&1
done
AN5D_LIB=paper_2001_01473_b200/libAN5D_seam.so timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "star2d1r or box2d1r or box2d2r or star2d2r or runs" > gpurun_out/pytest15_seam.log 2>&1
echo rc=$? >> gpurun_out/pytest15_seam.log
ls -la gpurun_out
