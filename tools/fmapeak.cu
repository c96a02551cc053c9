// FP32 / packed-FP32 / FP64 FMA-pipe peak microbenchmark (SURVEY N-6): many independent FMA chains
// per thread, full grid; prints GFLOP/s (2 flops per FMA lane).  Build: nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int CH = 16, IT = 4096;
__global__ void k_ffma(float* out, float c) {
    float a[CH];
    for (int j = 0; j < CH; ++j) a[j] = threadIdx.x + j;
    for (int i = 0; i < IT; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = fmaf(a[j], c, 0.5f);
    float s = 0; for (int j = 0; j < CH; ++j) s += a[j];
    if (s == 123.f) out[0] = s;
}
__global__ void k_ffma2(float* out, float c) {
    float2 a[CH];
    for (int j = 0; j < CH; ++j) a[j] = make_float2(threadIdx.x + j, j);
    const float2 cc = make_float2(c, c), h = make_float2(0.5f, 0.5f);
    for (int i = 0; i < IT; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = __ffma2_rn(a[j], cc, h);
    float s = 0; for (int j = 0; j < CH; ++j) s += a[j].x + a[j].y;
    if (s == 123.f) out[0] = s;
}
__global__ void k_dfma(float* out, double c) {
    double a[CH];
    for (int j = 0; j < CH; ++j) a[j] = threadIdx.x + j;
    for (int i = 0; i < IT; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = fma(a[j], c, 0.5);
    double s = 0; for (int j = 0; j < CH; ++j) s += a[j];
    if (s == 123.) out[0] = (float)s;
}
int main() {
    float* out; cudaMalloc(&out, 4);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = nsm * 8, thr = 256;
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) k_ffma<<<blocks, thr>>>(out, 0.999f);
            if (v == 1) k_ffma2<<<blocks, thr>>>(out, 0.999f);
            if (v == 2) k_dfma<<<blocks, thr>>>(out, 0.999);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double fmas = (double)blocks * thr * CH * IT * (v == 1 ? 2 : 1);
            if (rep == 2) printf("{\"kind\": \"%s\", \"gflops\": %.1f, \"ms\": %.3f}\n", v == 0 ? "ffma" : v == 1 ? "ffma2" : "dfma",
                                 2.0 * fmas / (ms * 1e-3) / 1e9, ms);
        }
    }
    return 0;
}
