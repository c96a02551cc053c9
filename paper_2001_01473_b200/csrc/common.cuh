// common.cuh -- small device helpers shared by the 2D and 3D N.5D kernels (sm_100a).
// Product code: never includes or links anything from oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>

namespace an5d {

// Cells per 16-byte vector: the B200 128-bit LDG/STG/LDS granule.
template <typename T> struct VecOf;
template <> struct VecOf<float> { using type = float4; static constexpr int A = 4; };
template <> struct VecOf<double> { using type = double2; static constexpr int A = 2; };

template <typename T>
__device__ __forceinline__ void ld_vec_global(T* dst, const T* src) {
    using V = typename VecOf<T>::type;
    V v = __ldg(reinterpret_cast<const V*>(src));
    if constexpr (VecOf<T>::A == 4) { dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w; }
    else { dst[0] = v.x; dst[1] = v.y; }
}

// Streamed-once loads: evict-first in L1 (the plane is consumed from registers; halo re-reads of
// neighbouring tiles hit L2).
template <typename T>
__device__ __forceinline__ void ld_vec_stream(T* dst, const T* src) {
    using V = typename VecOf<T>::type;
    V v = __ldcs(reinterpret_cast<const V*>(src));
    if constexpr (VecOf<T>::A == 4) { dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w; }
    else { dst[0] = v.x; dst[1] = v.y; }
}

template <typename T>
__device__ __forceinline__ void st_vec_global(T* dst, const T* src) {
    using V = typename VecOf<T>::type;
    V v;
    if constexpr (VecOf<T>::A == 4) { v.x = src[0]; v.y = src[1]; v.z = src[2]; v.w = src[3]; }
    else { v.x = src[0]; v.y = src[1]; }
    *reinterpret_cast<V*>(dst) = v;
}

template <typename T>
__device__ __forceinline__ void st_vec_shared(T* dst, const T* src) {
    using V = typename VecOf<T>::type;
    V v;
    if constexpr (VecOf<T>::A == 4) { v.x = src[0]; v.y = src[1]; v.z = src[2]; v.w = src[3]; }
    else { v.x = src[0]; v.y = src[1]; }
    *reinterpret_cast<V*>(dst) = v;
}

template <typename T>
__device__ __forceinline__ void ld_vec_shared(T* dst, const T* src) {
    using V = typename VecOf<T>::type;
    V v = *reinterpret_cast<const V*>(src);
    if constexpr (VecOf<T>::A == 4) { dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w; }
    else { dst[0] = v.x; dst[1] = v.y; }
}

// Non-negative modulo usable in constant expressions (static register-queue slots).
__host__ __device__ constexpr int pmod(int a, int m) { return ((a % m) + m) % m; }

// Coefficient storage in the kernel parameter space (constant bank 0): FFMA reads them as
// c[0x0][...] operands, so the taps cost no registers and no extra instructions.
template <typename T, int N> struct Coeffs { T c[N]; };

// Compile-time loop: f(integral_constant<int, I>) for I in [I0, N).
template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N>(f);
    }
}

}  // namespace an5d

namespace an5d {

// ---- cp.async (LDGSTS): 16-byte global -> shared copies, completion tracked per thread ----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Copies src_bytes (0..16) from gmem and zero-fills the rest of the 16-byte destination.
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
                 "r"(src_bytes));
}
// Predicated 16-byte copy (no branch: the predicate guards the instruction itself).
__device__ __forceinline__ void cp_async16_pred(void* sdst, const void* gsrc, int src_bytes, bool pred) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
                 " @p cp.async.cg.shared.global [%0], [%1], 16, %2;\n}\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
                 "r"(src_bytes), "r"((int)pred));
}
// Predicated element-sized copy (4 or 8 bytes, .ca) with zero-fill: src_bytes is 0 or N.
template <int N>
__device__ __forceinline__ void cp_async_elem_pred(void* sdst, const void* gsrc, int src_bytes, bool pred) {
    static_assert(N == 4 || N == 8, "cp.async.ca element size");
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                 " @p cp.async.ca.shared.global [%0], [%1], %2, %3;\n}\n" ::"r"(smem_u32(sdst)), "l"(gsrc), "n"(N),
                 "r"(src_bytes), "r"((int)pred));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace an5d
