// inst2d.cuh -- launcher and registry entry of one 2D kernel instance (included by the generated
// csrc/gen/inst_2d_*.cu files only, so a 2D change does not rebuild the 3D instances).
#pragma once
#include "kernel2d.cuh"
#include "registry.hpp"

namespace an5d {

template <typename T, int R, int BT, int V, bool BOX, bool ASSOC, int NW = 1, bool GRAD = false, int NF = 1>
cudaError_t launch2d(const Sweep2DArgs& a, const void* coeffs, int64_t blocks, bool /*edge*/,
                     cudaStream_t st) {
    Coeffs2D<T, R, NF> cf;
    const T* c0 = static_cast<const T*>(coeffs);
    constexpr int W = 2 * R + 1;
    constexpr int CB = W * W + W;   // parameter block per (output, input) field pair
    for (int b = 0; b < NF * NF; ++b) {   // host table: NF^2 dense W x W blocks, block i NF + j
        const T* c = c0 + b * W * W;
        for (int i = 0; i < W * W; ++i) {
            if constexpr (sizeof(T) == 4) cf.c[b * CB + i] = make_float2(c[i], c[i]);   // broadcast pair (FFMA2)
            else cf.c[b * CB + i] = c[i];
        }
        for (int dy = 0; dy < W; ++dy) {   // mixed pairs (c[dy][+1], c[dy][-1]) for the swapped FFMA2
            if constexpr (sizeof(T) == 4) cf.c[b * CB + W * W + dy] = make_float2(c[dy * W + R + 1], c[dy * W + R - 1]);
            else cf.c[b * CB + W * W + dy] = 0;
        }
    }
    if constexpr (GRAD) {   // gradient2d: c_0 follows the dense table (an5d_create)
        if constexpr (sizeof(T) == 4) cf.c[W * W] = make_float2(c0[W * W], c0[W * W]);
        else cf.c[W * W] = c0[W * W];
    }
    constexpr size_t smem = smem_bytes_2d<T, R, BT, V, ASSOC, NW, NF>();
    auto fn = &an5d_sweep2d<T, R, BT, V, BOX, ASSOC, NW, GRAD, NF>;
    static bool attr_set = false;   // once per instance (a per-launch attribute call costs host time)
    if (smem > 48 * 1024 && !attr_set) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set = true;
    }
    // programmatic dependent launch (common.cuh PDL): the kernel waits for the previous grid itself
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)blocks, 1, 1);
    lc.blockDim = dim3(32 * NW, 1, 1);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&lc, fn, a, cf);
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename T, int R, int BT, int V, bool BOX, bool ASSOC = true, int NW = 1, bool GRAD = false, int NF = 1>
Instance make_instance2d() {
    Instance i{};
    i.ndim = 2; i.shape = GRAD ? 2 : (BOX ? 1 : 0); i.dtype = sizeof(T) == 8 ? 1 : 0;
    i.rad = R; i.bT = BT; i.vec = V; i.assoc = ASSOC ? 1 : 0;
    i.launch2d = &launch2d<T, R, BT, V, BOX, ASSOC, NW, GRAD, NF>;
    i.nf = NF;
    i.launch3d = nullptr;
    i.fn_interior = reinterpret_cast<const void*>(&an5d_sweep2d<T, R, BT, V, BOX, ASSOC, NW, GRAD, NF>);
    i.fn_edge = i.fn_interior;
    i.threads = 32 * NW;
    i.tile_x_loaded = 32 * V;
    i.tile_y = 0;
    i.smem_bytes = smem_bytes_2d<T, R, BT, V, ASSOC, NW, NF>();
    return i;
}

}  // namespace an5d
