// registry.hpp -- table of compiled sm_100a kernel instances (filled by the generated inst_*.cu
// files at library load time).  A kernel instance is one specialisation of the N.5D sweep:
// (ndim, shape, dtype, rad, b_T, register tiling).  The paper generates one kernel per stencil and
// configuration at compile time; here the instances are compiled once and picked at
// run time by the host planner.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "args.hpp"

namespace an5d {

using Launch2DFn = cudaError_t (*)(const Sweep2DArgs&, const void* coeffs, int64_t blocks, bool edge,
                                   cudaStream_t);
using Launch3DFn = cudaError_t (*)(const Sweep3DArgs&, const void* coeffs, const CUtensorMap& tmap, int64_t blocks,
                                   cudaStream_t);

struct Instance {
    int ndim, shape, dtype, rad, bT, vec;   // vec: cells per lane along x (2D) / y (3D)
    int assoc;                               // 1: associative partial sums; 0: direct gather (2D)
    Launch2DFn launch2d;
    Launch3DFn launch3d;
    const void* fn_interior;                 // for cudaFuncGetAttributes / occupancy queries
    const void* fn_edge;
    int threads;                             // threads per block
    int tile_x_loaded;                       // cells per tile along x (loaded window)
    int tile_y;                              // 3D: cells per tile along y; 2D: 0
    size_t smem_bytes;                       // dynamic shared memory per block
    int cluster;                             // 3D: blocks per cluster along y (tile_y = cluster x block rows)
    int nf;                                  // fields advanced together (multi-field systems; 0/1 = one)
    int xstage;                              // 3D x-staged layouts: staged x halo cells per side (0: none)
    int xpair;                               // 3D: loaded x halo = b_T rad exactly (Kernel3DTraits::XPAIR)
};

std::vector<Instance>& registry();

struct Registrar {
    explicit Registrar(const Instance& i) { registry().push_back(i); }
};

}  // namespace an5d
