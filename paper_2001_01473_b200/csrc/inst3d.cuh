// inst3d.cuh -- launcher and registry entry of one 3D kernel instance (included by the generated
// csrc/gen/inst_3d_*.cu files only).
#pragma once
#include "kernel3d.cuh"
#include "registry.hpp"

namespace an5d {

template <typename T, int R, int BT, int VY, bool BOX, int TXT, int VX, int CL = 1, int OS = 0>
cudaError_t launch3d(const Sweep3DArgs& a, const void* coeffs, const CUtensorMap& tmap, int64_t blocks,
                     cudaStream_t st) {
    using K = Kernel3DTraits<T, R, BT, VY, TXT, VX, OS>;
    constexpr int N = (2 * R + 1) * (2 * R + 1) * (2 * R + 1);
    Coeffs3D<T, R> cf;
    const T* c = static_cast<const T*>(coeffs);
    for (int i = 0; i < N; ++i) {
        if constexpr (sizeof(T) == 4) cf.c[i] = make_float2(c[i], c[i]);   // broadcast pair (FFMA2)
        else cf.c[i] = c[i];
    }
    constexpr int W = 2 * R + 1;
    for (int r = 0; r < W * W; ++r) {   // mixed pairs (c[dz][dy][+1], c[dz][dy][-1]), r = (dz+R) W + (dy+R)
        if constexpr (sizeof(T) == 4) cf.c[N + r] = make_float2(c[r * W + R + 1], c[r * W + R - 1]);
        else cf.c[N + r] = 0;
    }
    auto fn = &an5d_sweep3d<T, R, BT, VY, BOX, TXT, VX, CL, OS>;
    static bool attr_set = false;   // once per instance (a per-launch attribute call costs host time)
    if (!attr_set) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::smem_total(CL));
        attr_set = true;
    }
    // one cluster of CL blocks per unit (NEXT N2: cluster halo sharing along y); programmatic
    // dependent launch (common.cuh PDL): the kernel waits for the previous grid itself
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)(blocks * CL), 1, 1);
    lc.blockDim = dim3(K::kThreads, 1, 1);
    lc.dynamicSmemBytes = K::smem_total(CL);
    lc.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if constexpr (CL > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = CL;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    lc.attrs = at;
    lc.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&lc, fn, a, cf, tmap);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename T, int R, int BT, int VY, bool BOX, int TXT = 16, int VX = 4, int CL = 1, int OS = 0>
Instance make_instance3d() {
    using K = Kernel3DTraits<T, R, BT, VY, TXT, VX, OS>;
    Instance i{};
    i.ndim = 3; i.shape = BOX ? 1 : 0; i.dtype = sizeof(T) == 8 ? 1 : 0;
    i.rad = R; i.bT = BT; i.vec = VY; i.assoc = 1;
    i.launch2d = nullptr;
    i.launch3d = &launch3d<T, R, BT, VY, BOX, TXT, VX, CL, OS>;
    i.fn_interior = reinterpret_cast<const void*>(&an5d_sweep3d<T, R, BT, VY, BOX, TXT, VX, CL, OS>);
    i.fn_edge = i.fn_interior;
    i.threads = K::kThreads;
    i.tile_x_loaded = K::kTXW;   // loaded window (output-stationary: compute width + 2 x halo)
    i.xpair = K::XPAIR ? 1 : 0;  // x halo b_T rad exactly; TMA box 2 XOFF cells wider (Kernel3DTraits)
    i.xstage = K::HXO;
    i.tile_y = K::kTYL * CL;   // a cluster's blocks form one tile of CL x kTY rows (OS: + 2 rad halo rows)
    i.cluster = CL;
    i.smem_bytes = K::smem_total(CL);
    return i;
}

}  // namespace an5d
