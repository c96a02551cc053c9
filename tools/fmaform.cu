// FMA-pipe rate per SASS operand form on B200 (sm_100a): which FFMA / FFMA2 encodings issue at
// full rate?  The 2D sweep's taps are FFMA2 with a constant-bank coefficient pair plus scalar
// FFMAs with a constant-bank coefficient (kernel2d.cuh tap_pm1).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fmaform tools/fmaform.cu
// Prints one JSON line per form: GFLOP/s (2 FLOP per FMA lane) and warp-instructions per SM-cycle
// equivalent (clock from cudaDevAttrClockRate).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int CH = 16, IT = 2048;

struct P { float c[8]; float2 c2[4]; };

// FFMA R, R, R, R (coefficient in a register)
__global__ void k_rrr(float* out, float c) {
    float a[CH], cr = c * 1.0001f + (float)threadIdx.x * 1e-9f;
    for (int j = 0; j < CH; ++j) a[j] = threadIdx.x + j;
    for (int i = 0; i < IT; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = fmaf(a[j], cr, a[(j + 1) % CH] * 0 + 0.25f * a[j]);
    float s = 0; for (int j = 0; j < CH; ++j) s += a[j];
    if (s == 123.f) out[0] = s;
}
// FFMA acc = c[bank] * x + acc : the stencil tap form (x, acc registers)
__global__ void k_rcr(float* out, const __grid_constant__ P p) {
    float a[CH], x[CH];
    for (int j = 0; j < CH; ++j) { a[j] = threadIdx.x + j; x[j] = j * 0.5f + threadIdx.x; }
    for (int i = 0; i < IT; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = fmaf(p.c[j & 7], x[j], a[j]);
    float s = 0; for (int j = 0; j < CH; ++j) s += a[j];
    if (s == 123.f) out[0] = s;
}
// FFMA acc = x * imm + acc
__global__ void k_rir(float* out, float unused) {
    float a[CH], x[CH];
    for (int j = 0; j < CH; ++j) { a[j] = threadIdx.x + j; x[j] = j * 0.5f + threadIdx.x; }
    for (int i = 0; i < IT; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = fmaf(0.999f, x[j], a[j]);
    float s = 0; for (int j = 0; j < CH; ++j) s += a[j];
    if (s == 123.f) out[0] = s;
}
// FFMA2 acc = c2[bank] * x + acc
__global__ void k_f2c(float* out, const __grid_constant__ P p) {
    float2 a[CH], x[CH];
    for (int j = 0; j < CH; ++j) { a[j] = make_float2(threadIdx.x + j, j); x[j] = make_float2(j * 0.5f, threadIdx.x); }
    for (int i = 0; i < IT; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = __ffma2_rn(p.c2[j & 3], x[j], a[j]);
    float s = 0; for (int j = 0; j < CH; ++j) s += a[j].x + a[j].y;
    if (s == 123.f) out[0] = s;
}
// FFMA2 with all-register operands
__global__ void k_f2r(float* out, float c) {
    float2 a[CH], x[CH];
    const float2 cc = make_float2(c * 1.0001f + threadIdx.x * 1e-9f, c);
    for (int j = 0; j < CH; ++j) { a[j] = make_float2(threadIdx.x + j, j); x[j] = make_float2(j * 0.5f, threadIdx.x); }
    for (int i = 0; i < IT; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = __ffma2_rn(cc, x[j], a[j]);
    float s = 0; for (int j = 0; j < CH; ++j) s += a[j].x + a[j].y;
    if (s == 123.f) out[0] = s;
}
// the 2D tap mix per cell pair: 4 FFMA2 (const pair) + 2 scalar FFMA (const)
__global__ void k_mix(float* out, const __grid_constant__ P p) {
    float2 a[CH / 2], x[CH / 2];
    for (int j = 0; j < CH / 2; ++j) { a[j] = make_float2(threadIdx.x + j, j); x[j] = make_float2(j * 0.5f, threadIdx.x); }
    for (int i = 0; i < IT; ++i)
#pragma unroll
        for (int j = 0; j < CH / 2; ++j) {
            a[j] = __ffma2_rn(p.c2[0], x[j], a[j]);
            a[j] = __ffma2_rn(p.c2[1], x[(j + 1) % (CH / 2)], a[j]);
            a[j] = __ffma2_rn(p.c2[2], x[(j + 2) % (CH / 2)], a[j]);
            a[j] = __ffma2_rn(p.c2[3], make_float2(x[j].y, x[j].x), a[j]);
            a[j].x = fmaf(p.c[0], x[(j + 3) % (CH / 2)].y, a[j].x);
            a[j].y = fmaf(p.c[1], x[(j + 5) % (CH / 2)].x, a[j].y);
        }
    float s = 0; for (int j = 0; j < CH / 2; ++j) s += a[j].x + a[j].y;
    if (s == 123.f) out[0] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    int nsm, khz;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    P p;
    for (int i = 0; i < 8; ++i) p.c[i] = 0.999f - i * 1e-4f;
    for (int i = 0; i < 4; ++i) p.c2[i] = make_float2(0.998f - i * 1e-4f, 0.997f);
    const int blocks = nsm * 8, thr = 256;
    const char* names[] = {"ffma_rrr", "ffma_const", "ffma_imm", "ffma2_const", "ffma2_rrr", "mix_4ffma2_2ffma"};
    for (int v = 0; v < 6; ++v) {
        float ms = 0;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) k_rrr<<<blocks, thr>>>(out, 0.999f);
            if (v == 1) k_rcr<<<blocks, thr>>>(out, p);
            if (v == 2) k_rir<<<blocks, thr>>>(out, 0.f);
            if (v == 3) k_f2c<<<blocks, thr>>>(out, p);
            if (v == 4) k_f2r<<<blocks, thr>>>(out, 0.999f);
            if (v == 5) k_mix<<<blocks, thr>>>(out, p);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        // FMA lanes per kernel
        double lanes = (double)blocks * thr * IT;
        double instr_per_thread_iter = v == 5 ? (CH / 2) * 6 : CH;
        double fma_lanes = v == 5 ? lanes * (CH / 2) * (4 * 2 + 2) : lanes * CH * (v >= 3 ? 2 : 1);
        double warp_instr = (double)blocks * thr / 32 * IT * instr_per_thread_iter;
        double sm_cycles = ms * 1e-3 * khz * 1e3;
        printf("{\"form\": \"%s\", \"gflops\": %.1f, \"ms\": %.3f, \"warp_instr_per_sm_cycle\": %.3f, "
               "\"fma_lanes_per_sm_cycle\": %.1f}\n",
               names[v], 2.0 * fma_lanes / (ms * 1e-3) / 1e9, ms, warp_instr / nsm / sm_cycles,
               fma_lanes / nsm / sm_cycles);
    }
    return 0;
}
