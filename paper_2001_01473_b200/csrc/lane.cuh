// lane.cuh -- register layout of one lane's V consecutive x cells in the 2D sweep (sm_100a).
//
// The stencil arithmetic works on "elements":
//   * fp64: one element = one cell (DFMA; the FP64 pipe is the bound, issue has slack);
//   * fp32: one element = a PAIR of adjacent cells (2e, 2e+1) in a float2, so the sm_100 packed
//     FFMA2/FMUL2 instructions do two cell updates per issue slot (measured: same FLOP/s as FFMA,
//     half the instructions -- tools/fmapeak.cu), freeing issue slots.  Taps whose x offset is
//     even (and every off-centre row tap of a star stencil) read an aligned pair; taps with an odd
//     x offset straddle two pairs and are done as two scalar FFMAs on the pair's halves (no
//     repacking moves).  The pair order equals the register order of LDS.128 / STG.128.
// The in-row halo (rad cells from each neighbouring lane) comes from 2*rad shuffles per level.
#pragma once
#include <cuda_runtime.h>

namespace an5d {

template <typename T, int V> struct Lane;

template <int V> struct Lane<double, V> {
    using E = double;
    static constexpr int NE = V;
    __device__ static __forceinline__ E fma(E c, E q, E acc) { return ::fma(c, q, acc); }
    __device__ static __forceinline__ E mul(E c, E q) { return c * q; }
    // cells <-> elements
    __device__ static __forceinline__ void from_cells(E (&P)[NE], const double (&c)[V]) {
#pragma unroll
        for (int v = 0; v < V; ++v) P[v] = c[v];
    }
    __device__ static __forceinline__ void to_cells(double (&c)[V], const E (&P)[NE]) {
#pragma unroll
        for (int v = 0; v < V; ++v) c[v] = P[v];
    }
    __device__ static __forceinline__ double& cell(E (&P)[NE], int v) { return P[v]; }
    __device__ static __forceinline__ double cell(const E (&P)[NE], int v) { return P[v]; }
};

template <int V> struct Lane<float, V> {
    using E = float2;
    static constexpr int NE = V / 2;
    static_assert(V % 2 == 0, "fp32 lanes hold pairs");
    __device__ static __forceinline__ E fma(E c, E q, E acc) { return __ffma2_rn(c, q, acc); }
    __device__ static __forceinline__ E mul(E c, E q) { return __fmul2_rn(c, q); }
    // element e = cells (2e, 2e+1): the register order of LDS.128 / STG.128, so no repacking
    __device__ static __forceinline__ void from_cells(E (&P)[NE], const float (&c)[V]) {
#pragma unroll
        for (int e = 0; e < NE; ++e) P[e] = make_float2(c[2 * e], c[2 * e + 1]);
    }
    __device__ static __forceinline__ void to_cells(float (&c)[V], const E (&P)[NE]) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            c[2 * e] = P[e].x;
            c[2 * e + 1] = P[e].y;
        }
    }
    __device__ static __forceinline__ float& cell(E (&P)[NE], int v) { return (v & 1) ? P[v >> 1].y : P[v >> 1].x; }
    __device__ static __forceinline__ float cell(const E (&P)[NE], int v) { return (v & 1) ? P[v >> 1].y : P[v >> 1].x; }
};

// coefficient as an element (fp32: broadcast pair, pre-duplicated in the parameter table)
template <typename T> struct CoefElem { using type = T; };
template <> struct CoefElem<float> { using type = float2; };

}  // namespace an5d
