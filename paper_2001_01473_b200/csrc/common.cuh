// common.cuh -- small device helpers shared by the 2D and 3D N.5D kernels (sm_100a).
// Product code: never includes or links anything from oracle/.
#pragma once
#include <cstdint>
#include <cstdlib>
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

// ---- programmatic dependent launch (PDL) between consecutive sweeps ------------------------------
// A sweep launched with cudaLaunchAttributeProgrammaticStreamSerialization may be scheduled while
// the previous sweep on the stream is still draining its last units; every sweep kernel therefore
// starts with pdl_wait() (griddepcontrol.wait: blocks until the previous grid has COMPLETED and its
// memory is visible -- before any global read or write, so the in-place buffer reuse of the sweep
// schedule stays ordered) and then pdl_trigger() (lets the NEXT sweep's blocks be scheduled onto
// SMs this grid frees).  Trigger after wait, never before: a grid two launches ahead holding SM
// slots while this one still needs them could deadlock.  Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
// host: PDL only with AN5D_PDL=1 (read once).  Off by default: at a fixed configuration the
// headline run measured 0.4 % SLOWER with it (3744-3753 vs 3761-3768 GCells/s, 4 interleaved runs
// each, profiles/r02pdl2_*); the kernels keep the wait / trigger (no-ops without the attribute)
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("AN5D_PDL");
        return e && e[0] == '1';
    }();
    return on;
}

// ---- TMA (cp.async.bulk.tensor) + mbarrier: whole tile planes staged by one thread ---------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// Block until phase `parity` of the barrier has completed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile("{\n .reg .pred done;\n"
                 "WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
                 " @!done bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
                 : "memory");
}
// 3D tiled TMA load of box {x, y, z} at coordinates (c0 = x, c1 = y, c2 = z) into shared memory;
// out-of-bound elements (negative or past the tensor's dims) are zero-filled by the hardware.
__device__ __forceinline__ void tma_load_3d(void* sdst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(sdst)),
                 "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
                 : "memory");
}
// ---- thread-block clusters (DSMEM) -------------------------------------------------------------
__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
// barrier over every thread of the cluster; release/acquire at cluster scope orders the shared
// memory writes before it with the (local or remote) reads after it
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// split-phase cluster barrier: arrive (release: this thread's prior shared-memory writes become
// visible to the cluster) ... independent work ... wait (acquire)
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// generic address of the same shared-memory location in CTA `rank` of the cluster (DSMEM):
// ordinary loads through it read the peer's shared memory
template <typename T>
__device__ __forceinline__ const T* map_cta(const T* p, unsigned rank) {
    uint64_t out;
    asm volatile("mapa.u64 %0, %1, %2;\n" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
    return reinterpret_cast<const T*>(out);
}

__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

}  // namespace an5d
