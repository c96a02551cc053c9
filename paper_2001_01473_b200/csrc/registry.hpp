// registry.hpp -- table of compiled sm_100a kernel instances (filled by the generated inst_*.cu
// files at library load time).  A kernel instance is one specialisation of the N.5D sweep:
// (ndim, shape, dtype, rad, b_T, register tiling).  The paper generates one kernel per stencil and
// configuration at compile time; here the instances are compiled once and picked at
// run time by the host planner.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "kernel2d.cuh"
#include "kernel3d.cuh"

namespace an5d {

using Launch2DFn = cudaError_t (*)(const Sweep2DArgs&, const void* coeffs, int64_t blocks, bool edge,
                                   cudaStream_t);
using Launch3DFn = cudaError_t (*)(const Sweep3DArgs&, const void* coeffs, int64_t blocks, bool edge,
                                   cudaStream_t);

struct Instance {
    int ndim, shape, dtype, rad, bT, vec;   // vec: cells per lane along x (2D) / y (3D)
    Launch2DFn launch2d;
    Launch3DFn launch3d;
    const void* fn_interior;                 // for cudaFuncGetAttributes / occupancy queries
    const void* fn_edge;
    int threads;                             // threads per block
    int tile_x_loaded;                       // cells per tile along x (loaded window)
    int tile_y;                              // 3D: cells per tile along y; 2D: 0
    size_t smem_bytes;                       // dynamic shared memory per block
};

std::vector<Instance>& registry();

struct Registrar {
    explicit Registrar(const Instance& i) { registry().push_back(i); }
};

template <typename T, int R, int BT, int V, bool BOX>
cudaError_t launch2d(const Sweep2DArgs& a, const void* coeffs, int64_t blocks, bool /*edge*/,
                     cudaStream_t st) {
    Coeffs2D<T, R> cf;
    const T* c = static_cast<const T*>(coeffs);
    for (int i = 0; i < (2 * R + 1) * (2 * R + 1); ++i) {
        if constexpr (sizeof(T) == 4) cf.c[i] = make_float2(c[i], c[i]);   // broadcast pair (FFMA2)
        else cf.c[i] = c[i];
    }
    constexpr size_t smem = smem_bytes_2d<T, R, BT, V>();
    auto fn = &an5d_sweep2d<T, R, BT, V, BOX>;
    static bool attr_set = false;   // once per instance (a per-launch attribute call costs host time)
    if (smem > 48 * 1024 && !attr_set) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set = true;
    }
    fn<<<(unsigned)blocks, 32, smem, st>>>(a, cf);
    return cudaGetLastError();
}

template <typename T, int R, int BT, int V, bool BOX>
Instance make_instance2d() {
    Instance i{};
    i.ndim = 2; i.shape = BOX ? 1 : 0; i.dtype = sizeof(T) == 8 ? 1 : 0;
    i.rad = R; i.bT = BT; i.vec = V;
    i.launch2d = &launch2d<T, R, BT, V, BOX>;
    i.launch3d = nullptr;
    i.fn_interior = reinterpret_cast<const void*>(&an5d_sweep2d<T, R, BT, V, BOX>);
    i.fn_edge = i.fn_interior;
    i.threads = 32;
    i.tile_x_loaded = 32 * V;
    i.tile_y = 0;
    i.smem_bytes = smem_bytes_2d<T, R, BT, V>();
    return i;
}

template <typename T, int R, int BT, int VY, bool BOX>
cudaError_t launch3d(const Sweep3DArgs& a, const void* coeffs, int64_t blocks, bool /*edge*/,
                     cudaStream_t st) {
    using K = Kernel3DTraits<T, R, BT, VY>;
    constexpr int N = (2 * R + 1) * (2 * R + 1) * (2 * R + 1);
    Coeffs3D<T, R> cf;
    const T* c = static_cast<const T*>(coeffs);
    for (int i = 0; i < N; ++i) {
        if constexpr (sizeof(T) == 4) cf.c[i] = make_float2(c[i], c[i]);   // broadcast pair (FFMA2)
        else cf.c[i] = c[i];
    }
    auto fn = &an5d_sweep3d<T, R, BT, VY, BOX>;
    static bool attr_set = false;   // once per instance (a per-launch attribute call costs host time)
    if (!attr_set) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::kSmemBytes);
        attr_set = true;
    }
    fn<<<(unsigned)blocks, K::kThreads, K::kSmemBytes, st>>>(a, cf);
    return cudaGetLastError();
}

template <typename T, int R, int BT, int VY, bool BOX>
Instance make_instance3d() {
    using K = Kernel3DTraits<T, R, BT, VY>;
    Instance i{};
    i.ndim = 3; i.shape = BOX ? 1 : 0; i.dtype = sizeof(T) == 8 ? 1 : 0;
    i.rad = R; i.bT = BT; i.vec = VY;
    i.launch2d = nullptr;
    i.launch3d = &launch3d<T, R, BT, VY, BOX>;
    i.fn_interior = reinterpret_cast<const void*>(&an5d_sweep3d<T, R, BT, VY, BOX>);
    i.fn_edge = i.fn_interior;
    i.threads = K::kThreads;
    i.tile_x_loaded = K::kTX;
    i.tile_y = K::kTY;
    i.smem_bytes = K::kSmemBytes;
    return i;
}

}  // namespace an5d
