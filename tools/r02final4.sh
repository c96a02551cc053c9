# round 2 final evidence (r02final4) at HEAD: smoke, default bench, reference arm, ncu launch list +
# full capture of the headline sweep, the whole suite (all Table-2 stencils fp32/fp64, systems, config 4)
NCU_CASE="star2d1r f32 8 45 8 6 32" bash tools/gpu_check.sh r02final4 smoke bench reference ncu suite
