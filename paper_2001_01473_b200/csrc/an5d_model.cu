// an5d_model.cu -- the paper's section-5 performance model and its "Tuned" search
// space, as pure host arithmetic behind the C ABI (include/an5d.h).  Product code:
// shares nothing with oracle/.
//
// Reading of the under-specified thread census:
//   * one cell per thread, n_thr = prod b_S_i threads per block;
//   * per (tile, stream block): level T = 1..bT computes on its valid region
//     prod (b_S_i - 2 T rad) over h + 2 rad (bT - T) planes (the stream-block overlap,
//     P:427-429) and reads shared memory there (Table 3 "practical" reads);
//   * every thread writes one shared-memory cell per plane at levels 0..bT-1 (even
//     out-of-bound threads write), over the same plane counts;
//   * global memory: one read per thread and plane at T = 0 over h + 2 bT rad planes, one write
//     per compute-region cell and plane at T = bT;
//   * FLOPs per computing thread-level = Table 2's FLOP/cell; eff_ALU with k-1 FMA +
//     1 MUL (+1 MUL for the j-stencil division under fast math);
//   * eff_SM = floor(w) / ceil(w), w = n'_tb / (n_SM * floor(2048 / n_thr)) (the
//     printed formula omits n_SM, which the same paragraph defines -- reading C-12).
// With Table 4's V100 numbers this reproduces Table 5's "Model" column within +-15 % on 15/20
// single- and 14/20 double-precision rows (tests/test_model_paper.py), and Table 5's tuned
// configuration is among the model's top 5 for 31 of the 40 rows (P:784-793 picks the measured
// best of the model's top 5).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/an5d.h"

namespace an5d {
an5d_status set_error(an5d_status s, const char* msg);   // an5d_host.cu (thread-local message)
}

namespace {

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

an5d_status model_eval(int ndim, int rad, an5d_shape shape, int has_div, an5d_dtype dtype, const int64_t* I,
                       int bT, const int* bS, int64_t h, const an5d_device_params& dev, an5d_model_result& r) {
    const int nb = ndim - 1;
    const int w = 2 * rad + 1;
    const int taps = shape == AN5D_BOX ? (ndim == 2 ? w * w : w * w * w) : 2 * ndim * rad + 1;
    const double F = 2.0 * taps - 1 + (has_div ? 1 : 0);                      // Table 2
    const double n_fma = taps - 1, n_mul = 1 + (has_div ? 1 : 0);
    const double eff_alu = (2 * n_fma + n_mul) / (2 * (n_fma + n_mul));
    // Table 3 practical shared-memory reads per computing thread and level
    double sm_reads;
    if (shape == AN5D_STAR) sm_reads = ndim == 2 ? 2.0 * rad : 4.0 * rad;
    else sm_reads = ndim == 2 ? (double)w - 1 : (double)w * w - 1;
    int64_t n_thr = 1, C[2] = {0, 0};
    for (int i = 0; i < nb; ++i) {
        C[i] = (int64_t)bS[i] - 2LL * bT * rad;
        if (C[i] < 1) return AN5D_ERR_INFEASIBLE_CONFIG;
        n_thr *= bS[i];
    }
    if (n_thr > dev.max_threads_per_sm) return AN5D_ERR_INFEASIBLE_CONFIG;
    int64_t n_tb = 1;
    for (int i = 0; i < nb; ++i) n_tb *= cdiv(I[1 + i], C[i]);
    const int64_t n_sb = cdiv(I[0], h);
    const int64_t n_tbp = n_tb * n_sb;
    double comp = 0, smr = 0, smw = 0;
    for (int T = 1; T <= bT; ++T) {
        double valid = 1;
        for (int i = 0; i < nb; ++i) valid *= (double)(bS[i] - 2 * T * rad);
        const double planes = (double)h + 2.0 * rad * (bT - T);
        comp += valid * planes;
        smr += valid * planes * sm_reads;
    }
    for (int T = 0; T < bT; ++T) smw += (double)n_thr * ((double)h + 2.0 * rad * (bT - T));
    const double gmr = (double)n_thr * ((double)h + 2.0 * bT * rad);
    double gmw = (double)h;
    for (int i = 0; i < nb; ++i) gmw *= (double)C[i];
    const double nw = dtype == AN5D_F32 ? 4.0 : 8.0;
    r.th_comp = comp * n_tbp;
    r.th_sm_read = smr * n_tbp;
    r.th_sm_write = smw * n_tbp;
    r.th_gm_read = gmr * n_tbp;
    r.th_gm_write = gmw * n_tbp;
    r.n_tb = n_tb;
    r.n_tb_prime = n_tbp;
    r.n_thr = (int)n_thr;
    r.flops_per_cell = F;
    r.eff_alu = eff_alu;
    r.time_comp = r.th_comp * F / (dev.peak_comp_gflops * 1e9 * eff_alu);
    r.time_sm = (r.th_sm_read + r.th_sm_write) * nw / (dev.peak_sm_gbs * 1e9);
    r.time_gm = (r.th_gm_read + r.th_gm_write) * nw / (dev.peak_gm_gbs * 1e9);
    const double cap = (double)dev.n_sm * (double)(dev.max_threads_per_sm / n_thr);
    const double waves = (double)n_tbp / cap;
    r.eff_sm = waves >= 1.0 ? std::floor(waves) / std::ceil(waves) : waves;   // < 1 wave: fraction used
    const double tmax = std::max(r.time_comp, std::max(r.time_sm, r.time_gm));
    r.bottleneck = tmax == r.time_comp ? 0 : (tmax == r.time_sm ? 1 : 2);
    r.time_model = tmax / r.eff_sm;
    double cells = 1;
    for (int i = 0; i < ndim; ++i) cells *= (double)I[i];
    r.gflops = cells * bT * F / r.time_model / 1e9;
    return AN5D_OK;
}

an5d_status check_args(int ndim, int radius, an5d_shape shape, an5d_dtype dtype, const int64_t* interior,
                       const an5d_device_params* dev) {
    if (ndim != 2 && ndim != 3) return AN5D_ERR_INVALID_ARGUMENT;
    if (radius < 1 || radius > 4) return AN5D_ERR_INVALID_ARGUMENT;
    if (shape != AN5D_STAR && shape != AN5D_BOX) return AN5D_ERR_INVALID_ARGUMENT;
    if (dtype != AN5D_F32 && dtype != AN5D_F64) return AN5D_ERR_INVALID_ARGUMENT;
    if (!interior || !dev) return AN5D_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < ndim; ++i)
        if (interior[i] < 1) return AN5D_ERR_INVALID_ARGUMENT;
    if (dev->n_sm < 1 || dev->max_threads_per_sm < 32 || !(dev->peak_comp_gflops > 0) || !(dev->peak_gm_gbs > 0) ||
        !(dev->peak_sm_gbs > 0))
        return AN5D_ERR_INVALID_ARGUMENT;
    return AN5D_OK;
}

}  // namespace

extern "C" {

an5d_status an5d_model_paper(int ndim, int radius, an5d_shape shape, int has_divisor, an5d_dtype dtype,
                             const int64_t* interior, int bT, const int* bS, int64_t h,
                             const an5d_device_params* dev, an5d_model_result* out) {
    an5d_status s = check_args(ndim, radius, shape, dtype, interior, dev);
    if (s != AN5D_OK || !out || !bS || bT < 1 || h < 1)
        return an5d::set_error(AN5D_ERR_INVALID_ARGUMENT, "an5d_model_paper: bad argument");
    an5d_model_result r{};
    s = model_eval(ndim, radius, shape, has_divisor, dtype, interior, bT, bS, h, *dev, r);
    if (s != AN5D_OK) return an5d::set_error(s, "an5d_model_paper: b_S - 2 bT rad < 1 or too many threads");
    *out = r;
    return AN5D_OK;
}

an5d_status an5d_model_paper_search(int ndim, int radius, an5d_shape shape, int has_divisor, an5d_dtype dtype,
                                    const int64_t* interior, const an5d_device_params* dev, int cap,
                                    an5d_config* out_cfg, double* out_gflops, int* n_feasible) {
    an5d_status s = check_args(ndim, radius, shape, dtype, interior, dev);
    if (s != AN5D_OK || cap < 0) return an5d::set_error(AN5D_ERR_INVALID_ARGUMENT, "an5d_model_paper_search: bad argument");
    struct Cand { double g; an5d_config c; };
    std::vector<Cand> all;
    const int bt_max = ndim == 2 ? 16 : 8;
    std::vector<std::pair<int, int>> tiles;      // {b_S_y, b_S_x}; 2D uses .second only
    std::vector<int64_t> hs;
    if (ndim == 2) {
        tiles = {{0, 128}, {0, 256}, {0, 512}};
        hs = {256, 512, 1024};
    } else {
        tiles = {{16, 16}, {16, 32}, {32, 32}, {16, 64}};   // "16x16, 32x16, 32x32, 64x16" (x x y)
        hs = {128, 256};
    }
    for (int bT = 1; bT <= bt_max; ++bT) {
        const int regs = dtype == AN5D_F32 ? bT * (2 * radius + 1) + bT + 20 : 2 * bT * (2 * radius + 1) + bT + 30;
        for (const auto& t : tiles) {
            const int bS[2] = {ndim == 2 ? t.second : t.first, t.second};
            const int64_t n_thr = ndim == 2 ? t.second : (int64_t)t.first * t.second;
            if (regs > 255 || regs * n_thr > 65536) continue;     // P:778-784 pruning
            for (int64_t h : hs) {
                an5d_model_result r{};
                if (model_eval(ndim, radius, shape, has_divisor, dtype, interior, bT, bS, h, *dev, r) != AN5D_OK)
                    continue;
                an5d_config c{};
                c.bT = bT;
                c.h = h;
                if (ndim == 2) { c.bS[0] = bS[0]; c.bS[1] = 0; }
                else { c.bS[0] = bS[0]; c.bS[1] = bS[1]; }
                all.push_back({r.gflops, c});
            }
        }
    }
    std::stable_sort(all.begin(), all.end(), [](const Cand& a, const Cand& b) { return a.g > b.g; });
    if (n_feasible) *n_feasible = (int)all.size();
    for (int i = 0; i < cap && i < (int)all.size(); ++i) {
        if (out_cfg) out_cfg[i] = all[i].c;
        if (out_gflops) out_gflops[i] = all[i].g;
    }
    return AN5D_OK;
}

}  // extern "C"
