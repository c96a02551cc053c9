// an5d_host.cu -- libAN5D host side: C ABI (include/an5d.h), sweep geometry, sweep schedule,
// B200 planner, launch orchestration.  Product code: shares nothing with oracle/.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>   // PFN_cuTensorMapEncodeTiled (driver entry point, no libcuda link)
#include <dlfcn.h>
#include <nccl.h>           // types only: NCCL is loaded at run time (an5d_set_comm)

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/an5d.h"
#include "registry.hpp"

namespace an5d {

std::vector<Instance>& registry() {
    static std::vector<Instance> r;
    return r;
}

namespace {

thread_local std::string g_err;

an5d_status fail(an5d_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

an5d_status cuda_fail(cudaError_t e, const char* where) {
    return fail(AN5D_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t round_up(int64_t a, int64_t m) { return cdiv(a, m) * m; }

}  // namespace

an5d_status set_error(an5d_status s, const char* msg) {
    g_err = msg;
    return s;
}

// ---------------------------------------------------------------------------------------------
// Plan
// ---------------------------------------------------------------------------------------------
struct Plan {
    int ndim, rad, shape, dtype;
    int nf = 1;                        // fields advanced together (an5d_create_system; NEXT N4)
    // NCCL slab mode (an5d_set_comm): this rank's slab of the streaming dimension
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1, ghost = 0;
    int64_t gE0 = 0, outer_offset = 0;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_bnd = nullptr, ev_xchg = nullptr;
    size_t elem;                       // bytes per cell (n_word)
    std::vector<double> coeffs_folded; // dense table / divisor (P:596-602 reciprocal folding)
    std::vector<unsigned char> coeffs_dev_t;  // rounded to dtype, as raw bytes
    double divisor;
    int device = -1;
    int64_t launches = 0;
    unsigned long long* ctr = nullptr;  // kCtrRing dynamic-scheduling counter pairs (device, zeroed)
    int64_t ctr_seq = 0;                // launches that used a counter pair
    // 2D run tables (device, immutable once built), keyed by the sweep geometry they schedule
    std::map<std::vector<int64_t>, std::pair<int4*, int64_t>> runs;
};
constexpr int kCtrRing = 64;            // counter pairs in flight per plan (>= concurrent sweeps)
constexpr int kScratch2D = 1024 * 32;   // Sweep2DArgs::scratch slots
constexpr size_t kRunCache = 64;        // run tables kept per plan

}  // namespace an5d

struct an5d_plan : an5d::Plan {};

namespace an5d {
namespace {

// ---------------------------------------------------------------------------------------------
// Sweep schedule (P:432-441 with DESIGN.md reading R-7)
//   degrees = [bT] * floor(T/bT) (+ [T mod bT]).  The result must land in grid_out after an odd
//   number of sweeps (each sweep flips the buffers, as the paper's (t+1)%2 indexing does).  If the
//   count is even, split the LAST sweep of degree >= 2 into (ceil(d/2), floor(d/2)) in place; if
//   every degree is 1 (bT == 1), append an interior copy instead.
// ---------------------------------------------------------------------------------------------
void make_schedule(int64_t T, int bT, std::vector<int>& deg, bool& trailing_copy) {
    deg.clear();
    trailing_copy = false;
    if (T <= 0) return;
    for (int64_t i = 0; i < T / bT; ++i) deg.push_back(bT);
    if (T % bT) deg.push_back((int)(T % bT));
    if (deg.size() % 2 == 0) {
        for (int64_t i = (int64_t)deg.size() - 1; i >= 0; --i) {
            if (deg[i] >= 2) {
                const int d = deg[i];
                deg[i] = (d + 1) / 2;
                deg.insert(deg.begin() + i + 1, d / 2);
                return;
            }
        }
        trailing_copy = true;
    }
}

// Kernel instance for (b_T, vec, direct) with a loaded tile width `tile_x` (0 = any) and
// `n_thr` threads per block (0 = any).  Among several matches the narrowest tile with the fewest
// threads is the default (the round-1 layouts), so a config that names neither keeps them.
const Instance* find_instance(const Plan& p, int bT, int vec, int direct = 0, int tile_x = 0, int n_thr = 0,
                              int tile_y = 0) {
    const Instance* best = nullptr;
    for (const Instance& i : registry())
        if (i.ndim == p.ndim && i.shape == p.shape && i.dtype == p.dtype && i.rad == p.rad && i.bT == bT &&
            i.vec == vec && i.assoc == (direct ? 0 : 1) && (!tile_x || i.tile_x_loaded == tile_x) &&
            (!n_thr || i.threads == n_thr) && (!tile_y || i.tile_y == tile_y) && std::max(1, i.nf) == p.nf)
            if (!best || std::make_tuple(i.tile_x_loaded, i.threads, i.tile_y) <
                             std::make_tuple(best->tile_x_loaded, best->threads, best->tile_y))
                best = &i;
    return best;
}

// Logical x tile b_S (compute region + 2 b_T rad) of an instance at full degree bT:
// what a configuration's bS names.  The loaded width minus the loaded halo (whole 16-byte vectors;
// x-staged 3D layouts: staged vectors + (b_T - 1) rad rounded) plus 2 b_T rad.
// 3D layouts without x staging hold a loaded x halo of exactly d rad (not rounded to a 16-byte
// vector) when fp32 and d rad = 2 mod 4 (kernel3d.cuh Kernel3DTraits::XPAIR; the instance of
// degree d carries the same decision in Instance::xpair, checked in sweep_geometry).
bool xpair_rule(const Plan& p, const Instance& i, int d) {
    return p.ndim == 3 && !i.xstage && p.elem == 4 && (d * p.rad) % 4 == 2;
}

// loaded x halo of instance i's layout at degree d
int x_halo(const Plan& p, const Instance& i, int d) {
    const int A = (int)(16 / p.elem), R = p.rad;
    if (p.ndim == 3 && i.xstage) return i.xstage + (int)round_up((int64_t)(d - 1) * R, A);
    return xpair_rule(p, i, d) ? d * R : (int)round_up((int64_t)d * R, A);
}

int inst_logical_x(const Plan& p, const Instance& i, int bT) {
    return i.tile_x_loaded - 2 * x_halo(p, i, bT) + 2 * bT * p.rad;
}

// Does instance i run degree-d sweeps of configuration c's layout?  The layout is named by
// (vec, direct, threads per block, logical b_S -- x through inst_logical_x at c's b_T, 3D y = the
// loaded height: the y halo is not rounded) -- fields left 0 match anything.
bool inst_matches(const Plan& p, const Instance& i, int d, const an5d_config& c, bool any_threads) {
    if (!(i.ndim == p.ndim && i.shape == p.shape && i.dtype == p.dtype && i.rad == p.rad && i.bT == d &&
          i.vec == c.vec && i.assoc == (c.direct ? 0 : 1) && std::max(1, i.nf) == p.nf))
        return false;
    if (!any_threads && c.n_thr && i.threads != c.n_thr) return false;
    const int bx = c.bS[p.ndim - 2];
    if (bx && c.bT && inst_logical_x(p, i, c.bT) != bx) return false;
    if (p.ndim == 3 && c.bS[0] && i.tile_y != c.bS[0]) return false;
    return true;
}

// The instance a sweep of degree d runs under configuration c: the configuration's layout, or for
// a reduced degree (d < b_T) without that layout (the 2D level split needs d >= 2) the same tile
// with any thread count -- identical per-cell arithmetic, so the results are the same bits.  Among
// several matches the narrowest tile with the fewest threads is the default (the round-1 layouts).
const Instance* find_instance(const Plan& p, int d, const an5d_config& c) {
    for (bool any : {false, true}) {
        if (any && d >= c.bT) break;
        const Instance* best = nullptr;
        for (const Instance& i : registry())
            if (inst_matches(p, i, d, c, any) &&
                (!best || std::make_tuple(i.tile_x_loaded, i.threads, i.tile_y) <
                              std::make_tuple(best->tile_x_loaded, best->threads, best->tile_y)))
                best = &i;
        if (best) return best;
    }
    return nullptr;
}

int max_bT_for(const Plan& p, int vec) {
    int m = 0;
    for (const Instance& i : registry())
        if (i.ndim == p.ndim && i.shape == p.shape && i.dtype == p.dtype && i.rad == p.rad &&
            i.vec == vec && std::max(1, i.nf) == p.nf)
            m = std::max(m, i.bT);
    return m;
}

// Sizes of the local problem
struct Dims {
    int64_t E[3];      // extents outer..x (ndim entries used)
    int64_t pitch[2];  // outer strides (2D: pitch[0] = row; 3D: pitch[0] = plane, pitch[1] = row)
    int64_t fstride = 0;  // multi-field systems: elements from one field's array to the next
};

// ---------------------------------------------------------------------------------------------
// Geometry of one sweep of degree d (bit-exact bookkeeping)
// ---------------------------------------------------------------------------------------------
struct SweepGeom {
    int A;                 // cells per 16-byte vector
    int loaded[2];         // loaded tile per blocked dim (outer..x)
    int halo[2];           // loaded halo per side
    int C[2];              // compute region per blocked dim
    int64_t ntiles[2];
    int64_t h, n_sb;
    // interior rectangle / box
    int64_t sb_lo, sb_hi;
    int64_t t_lo[2], t_hi[2];
    int64_t n_units, n_interior;
};

an5d_status sweep_geometry(const Plan& p, const Instance& inst, const Dims& dm, int d, int64_t h,
                           int64_t g_off, int64_t gE0, int64_t out_lo, int64_t out_hi, SweepGeom& g) {
    const int R = p.rad;
    g.A = (int)(16 / p.elem);
    const int nb = p.ndim - 1;  // blocked dims
    int loaded[2], halo[2];
    if (p.ndim == 2) {
        loaded[0] = inst.tile_x_loaded;
        halo[0] = (int)round_up((int64_t)d * R, g.A);
    } else {
        loaded[0] = inst.tile_y;
        halo[0] = d * R;
        loaded[1] = inst.tile_x_loaded;
        // x-staged layouts (kernel3d.cuh OS bit 1): the staged vectors beyond the threads plus the
        // (d-1) rad the threads' level-1 values shrink by, each rounded to whole vectors
        // (XPAIR layouts: exactly d rad; the host rule and the compiled instance must agree)
        if (xpair_rule(p, inst, d) != (inst.xpair != 0))
            return fail(AN5D_ERR_UNSUPPORTED, "instance x-halo rule mismatch (degree %d)", d);
        halo[1] = x_halo(p, inst, d);
    }
    for (int i = 0; i < nb; ++i) {
        g.loaded[i] = loaded[i];
        g.halo[i] = halo[i];
        g.C[i] = loaded[i] - 2 * halo[i];
        if (g.C[i] < 1)
            return fail(AN5D_ERR_INFEASIBLE_CONFIG,
                        "empty compute region: tile %d - 2*halo %d < 1 (P:320 b_S - 2 b_T rad >= 1)",
                        loaded[i], halo[i]);
        const int64_t I = dm.E[1 + i] - 2 * R;
        g.ntiles[i] = cdiv(I, g.C[i]);
        // interior tiles: loaded window [R + t C - H, +loaded) inside [R, E - R)
        const int64_t E = dm.E[1 + i];
        int64_t lo = 0, hi = g.ntiles[i];
        while (lo < hi && (R + lo * g.C[i] - halo[i] < R || R + lo * g.C[i] - halo[i] + loaded[i] > E - R)) ++lo;
        while (hi > lo && (R + (hi - 1) * g.C[i] - halo[i] + loaded[i] > E - R)) --hi;
        g.t_lo[i] = lo;
        g.t_hi[i] = hi;
    }
    const int64_t Iout = out_hi - out_lo;
    g.h = std::max<int64_t>(1, std::min<int64_t>(h, Iout));
    g.n_sb = cdiv(Iout, g.h);
    auto sb_edge = [&](int64_t sb) {
        const int64_t p0 = out_lo + sb * g.h, p1 = std::min(p0 + g.h, out_hi);
        const int64_t s0 = p0 - (int64_t)d * R, s1 = p1 + (int64_t)d * R;
        return s0 < 0 || s1 > dm.E[0] || s0 + g_off < R || s1 - 1 + g_off >= gE0 - R;
    };
    int64_t lo = 0, hi = g.n_sb;
    while (lo < hi && sb_edge(lo)) ++lo;
    while (hi > lo && sb_edge(hi - 1)) --hi;
    g.sb_lo = lo;
    g.sb_hi = hi;
    int64_t nt = 1, ni = hi - lo;
    for (int i = 0; i < nb; ++i) {
        nt *= g.ntiles[i];
        ni *= std::max<int64_t>(0, g.t_hi[i] - g.t_lo[i]);
    }
    // an empty interior box: everything is edge
    bool empty = (hi <= lo);
    for (int i = 0; i < nb; ++i) empty = empty || g.t_hi[i] <= g.t_lo[i];
    if (empty) {
        g.sb_lo = g.sb_hi = 0;
        for (int i = 0; i < nb; ++i) g.t_lo[i] = g.t_hi[i] = 0;
        ni = 0;
    }
    g.n_units = nt * g.n_sb;
    g.n_interior = ni;
    return AN5D_OK;
}

// ---------------------------------------------------------------------------------------------
// Device properties used by the planner
// ---------------------------------------------------------------------------------------------
struct DevInfo {
    int n_sm = 148;
    double clock_ghz = 1.965;
    double hbm_gbs = 6549.0;   // MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)
};

// Device properties and per-instance occupancy are queried once per device and cached: the
// runtime queries are not free (measured: a per-launch query made host-side launch gaps of
// tens of ms), and a sweep of T = 1000 steps issues hundreds of launches.
DevInfo dev_info() {
    static int cached_dev = -1;
    static DevInfo cached;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return DevInfo{}; }
    if (dev == cached_dev) return cached;
    DevInfo di;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) di.n_sm = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, dev) == cudaSuccess && v > 0) di.clock_ghz = v * 1e-6;
    cudaGetLastError();
    if (const char* e = getenv("AN5D_HBM_GBS")) di.hbm_gbs = atof(e);
    cached = di;
    cached_dev = dev;
    return di;
}

int resident_blocks(const Instance& inst) {
    static std::vector<std::pair<const void*, int>> cache;   // (kernel, blocks/SM); one device per process
    for (const auto& c : cache)
        if (c.first == inst.fn_interior) return c.second;
    int nblk = 0;
    if (inst.smem_bytes > 48 * 1024)
        cudaFuncSetAttribute(inst.fn_interior, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)inst.smem_bytes);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nblk, inst.fn_interior, inst.threads, inst.smem_bytes) !=
            cudaSuccess ||
        nblk < 1) {
        cudaGetLastError();
        nblk = 1;
    }
    cache.emplace_back(inst.fn_interior, nblk);
    return nblk;
}

// units resident on the whole GPU: resident blocks x SMs, divided by the blocks one unit takes
// (a 3D cluster layout runs one unit on CL blocks)
int64_t resident_units(const Instance& inst) {
    return std::max<int64_t>(1, (int64_t)resident_blocks(inst) * dev_info().n_sm / std::max(1, inst.cluster));
}

int taps_of(const Plan& p) {
    const int w = 2 * p.rad + 1;
    if (p.shape == AN5D_BOX) return p.ndim == 2 ? w * w : w * w * w;
    // gradient2d: 4 differences, 4 squares, 3 adds, c f + ..., and the IEEE sqrt and division
    // (each a MUFU seed plus ~8 FMA-pipe refinement ops): ~24 FMA-pipe ops per cell (R-17)
    if (p.shape == AN5D_GRADIENT) return 24;
    return p.ndim == 2 ? 4 * p.rad + 1 : 6 * p.rad + 1;
}

// 2D unit schedule ("runs").  A persistent warp that streams k consecutive stream blocks of one
// tile in a single pass pays the stream-block overlap (2 b_T rad rows) and the
// pipeline prologue once instead of k times; the output rows and their values are identical
// (every row is still produced by the same per-row arithmetic).  The table is handed out by the
// kernel's dynamic counter in this order:
//   1. x-edge tiles {0, nx-1, nx-2}: single stream blocks (slowest units first);
//   2. y-edge stream blocks (those touching the ring / array end) of the other tiles: singles;
//   3. one round of c = floor(W / n_interior_tiles) big runs per interior tile, k stream blocks
//      each, covering about `frac` of the y-interior stream blocks (W = launched warps, so every
//      warp gets about one big run);
//   4. the remaining y-interior stream blocks as singles: the dynamic tail balances on these.
// frac = AN5D_RUN_FRAC (default 0.85; 0 = singles only, the plain stream-block schedule).
std::vector<int4> build_runs_2d(const SweepGeom& g, int64_t W, double frac) {
    const int nx = (int)g.ntiles[0];
    const int nxe = nx < 4 ? nx : 3, ni = nx - nxe;
    std::vector<int4> r;
    r.reserve((size_t)(nx * g.n_sb));
    for (int64_t sb = 0; sb < g.n_sb; ++sb)
        for (int e = 0; e < nxe; ++e) r.push_back(make_int4(nx < 4 ? e : (e == 0 ? 0 : nx - e), (int)sb, (int)sb + 1, 0));
    if (ni == 0) return r;
    // y-interior stream blocks: the interior rectangle's range when it exists, else none
    int64_t lo = g.sb_lo, hi = g.sb_hi;
    if (hi <= lo) lo = hi = g.n_sb;
    for (int64_t sb = 0; sb < g.n_sb; ++sb)
        if (sb < lo || sb >= hi)
            for (int t = 1; t <= ni; ++t) r.push_back(make_int4(t, (int)sb, (int)sb + 1, 0));
    const int64_t nI = hi - lo;
    const int64_t c = std::max<int64_t>(1, W / ni);
    const int64_t k = (int64_t)(frac * (double)nI / (double)c);
    int64_t start = lo;
    if (k >= 2) {
        for (int64_t j = 0; j < c; ++j)
            for (int t = 1; t <= ni; ++t) r.push_back(make_int4(t, (int)(lo + j * k), (int)(lo + (j + 1) * k), 0));
        start = lo + c * k;
    }
    for (int64_t sb = start; sb < hi; ++sb)
        for (int t = 1; t <= ni; ++t) r.push_back(make_int4(t, (int)sb, (int)sb + 1, 0));
    return r;
}

// 3D: the same schedule over (tile y, tile x) with the kernel's frame-first order: frame tiles (first
// and last two in y and x: they may touch the ring and run the EDGE variant) as singles, z-edge
// stream blocks of interior tiles as singles, one round of long runs per interior tile, the rest as
// singles.  One thread block per entry, dispatched in index order by the hardware.
std::vector<int4> build_runs_3d(const SweepGeom& g, int64_t W, double frac) {
    const int ny = (int)g.ntiles[0], nx = (int)g.ntiles[1];
    auto frame = [&](int ty, int tx) { return ny < 4 || nx < 4 || ty == 0 || ty >= ny - 2 || tx == 0 || tx >= nx - 2; };
    std::vector<int4> r;
    std::vector<std::pair<int, int>> inner;
    for (int ty = 0; ty < ny; ++ty)
        for (int tx = 0; tx < nx; ++tx)
            if (!frame(ty, tx)) inner.emplace_back(ty, tx);
    r.reserve((size_t)(ny * nx * g.n_sb));
    for (int64_t sb = 0; sb < g.n_sb; ++sb)
        for (int ty = 0; ty < ny; ++ty)
            for (int tx = 0; tx < nx; ++tx)
                if (frame(ty, tx)) r.push_back(make_int4(ty, tx, (int)sb, (int)sb + 1));
    if (inner.empty()) return r;
    int64_t lo = g.sb_lo, hi = g.sb_hi;
    if (hi <= lo) lo = hi = g.n_sb;
    for (int64_t sb = 0; sb < g.n_sb; ++sb)
        if (sb < lo || sb >= hi)
            for (auto& t : inner) r.push_back(make_int4(t.first, t.second, (int)sb, (int)sb + 1));
    const int64_t ni = (int64_t)inner.size(), nI = hi - lo;
    const int64_t c = std::max<int64_t>(1, W / ni);
    const int64_t k = (int64_t)(frac * (double)nI / (double)c);
    int64_t start = lo;
    if (k >= 2) {
        for (int64_t j = 0; j < c; ++j)
            for (auto& t : inner) r.push_back(make_int4(t.first, t.second, (int)(lo + j * k), (int)(lo + (j + 1) * k)));
        start = lo + c * k;
    }
    for (int64_t sb = start; sb < hi; ++sb)
        for (auto& t : inner) r.push_back(make_int4(t.first, t.second, (int)sb, (int)sb + 1));
    return r;
}

// run table of a sweep geometry for W resident blocks (2D: persistent warps; 3D: blocks)
std::vector<int4> build_runs(int ndim, const SweepGeom& g, int64_t W, double frac) {
    return ndim == 2 ? build_runs_2d(g, W, frac) : build_runs_3d(g, W, frac);
}

double run_frac() {
    const char* e = getenv("AN5D_RUN_FRAC");   // read per call: tests switch it within a process
    return e ? std::max(0.0, std::min(0.98, atof(e))) : 0.85;
}

// warps the run table is shaped for: the launched persistent warps, or AN5D_RUN_WARPS (test knob:
// forces long runs on grids small enough for the oracle)
int64_t run_warps(int64_t blocks) {
    const char* e = getenv("AN5D_RUN_WARPS");
    return e && atoll(e) > 0 ? atoll(e) : blocks;
}

// Planner model: predicted seconds per cell-step of a configuration, in the
// spirit of the paper's section 5 model (one time per resource, the max of them, a
// waves efficiency) re-derived for this build's kernels on B200:
//   HBM term   bytes per sweep = loaded tile windows incl. halo and stream-block overlap (read) +
//              interior (written), / (measured copy bandwidth x eta_hbm);
//   FMA term   FMA-pipe operations per sweep = taps x every cell the kernel computes (the whole
//              loaded window at every level over h + 2 b_T rad (+ period) rows) /
//              (n_SM x FMA lanes x clock x eta_fma); FP64 has half the lanes;
//   tail       units are handed out dynamically, so the tail is about one unit: the time is
//              multiplied by (1 + resident / n_units)  (replaces eff_SM's wave quantisation).
// eta_* are the fractions of the measured peaks the kernels reach in steady state (tools/ runs
// on B200: star2d1r fp32 interior loop ~0.45 of the FMA peak; streaming at ~0.75 of copy BW).
double model_time(const Plan& p, const Instance& inst, const Dims& dm, int bT, int64_t h, const DevInfo& di,
                  SweepGeom* out_geom) {
    SweepGeom g{};
    if (sweep_geometry(p, inst, dm, bT, h, 0, dm.E[0], p.rad, dm.E[0] - p.rad, g) != AN5D_OK) return 1e30;
    const int R = p.rad;
    int64_t interior = 1;
    for (int i = 0; i < p.ndim; ++i) interior *= dm.E[i] - 2 * R;
    const int64_t rows_per_unit = g.h + 2LL * bT * R;
    int64_t cells_per_plane = 1;
    for (int i = 0; i < p.ndim - 1; ++i) cells_per_plane *= g.loaded[i];
    // steady-state fractions of the measured peaks the kernels reach on B200, per layout
    // (round 1-2 suites): 2D one warp per tile 0.45 of the FMA peak, the two-warp level split
    // 0.88x that; 3D 256-thread blocks 0.35, 512-thread fp64 blocks (twice the warps) 1.25x,
    // 512-thread fp32 128-wide tiles 0.87x
    const double eta_hbm = 0.75;
    double eta_fma = p.ndim == 2 ? 0.45 : 0.35;
    if (p.ndim == 2 && inst.threads == 64) eta_fma *= 0.88;
    if (p.ndim == 3 && inst.threads == 512) eta_fma *= p.dtype == AN5D_F64 ? 1.25 : 0.87;
    const double resident = (double)resident_units(inst);
    // units are runs of stream blocks (build_runs_2d / _3d); each run pays the overlap once
    double units = (double)g.n_units, unit_rows = (double)rows_per_unit;
    if (run_frac() > 0) {
        const double nt = (double)g.ntiles[0] * (p.ndim == 3 ? (double)g.ntiles[1] : 1.0);
        const int64_t W = p.ndim == 2 ? std::min<int64_t>(g.n_units, (int64_t)resident) : (int64_t)resident;
        units = (double)build_runs(p.ndim, g, W, run_frac()).size();
        unit_rows = nt * (double)(dm.E[0] - 2 * R) / units + 2.0 * bT * R;
    }
    const double bytes = (double)p.elem * p.nf * (units * unit_rows * cells_per_plane + (double)interior);
    const double t_hbm = bytes / (di.hbm_gbs * 1e9 * eta_hbm);
    const double fma_ops = units * (unit_rows + 2 * R + 1) * cells_per_plane * bT * taps_of(p) * p.nf * p.nf;
    const double lanes = p.dtype == AN5D_F64 ? 64.0 : 128.0;
    const double t_fma = fma_ops / (di.n_sm * lanes * di.clock_ghz * 1e9 * eta_fma);
    const double tail = 1.0 + resident / std::max<double>(1.0, (double)g.n_units);
    const double t = std::max(t_hbm, t_fma) * tail;
    if (out_geom) *out_geom = g;
    return t / ((double)interior * bT);
}

// Every feasible configuration with its model time (seconds per cell-step), best first.
std::vector<std::pair<double, an5d_config>> rank_configs(const Plan& p, const Dims& dm, int64_t T,
                                                         const an5d_config* hint) {
    const DevInfo di = dev_info();
    std::vector<std::pair<double, an5d_config>> out;
    const int64_t Iout = dm.E[0] - 2 * p.rad;
    for (const Instance& inst : registry()) {
        if (inst.ndim != p.ndim || inst.shape != p.shape || inst.dtype != p.dtype || inst.rad != p.rad ||
            std::max(1, inst.nf) != p.nf)
            continue;
        // gradient2d is non-associative: direct gather only
        const int direct = p.shape == AN5D_GRADIENT ? 1 : (hint ? hint->direct : 0);
        if (inst.assoc != (direct ? 0 : 1)) continue;
        if (hint && hint->bT && inst.bT != hint->bT) continue;
        if (hint && hint->vec && inst.vec != hint->vec) continue;
        if (hint && hint->n_thr && inst.threads != hint->n_thr) continue;
        if (hint && hint->bT && hint->bS[p.ndim - 2] && inst_logical_x(p, inst, hint->bT) != hint->bS[p.ndim - 2])
            continue;
        if (hint && p.ndim == 3 && hint->bS[0] && inst.tile_y != hint->bS[0]) continue;
        if (T > 0 && inst.bT > T) continue;
        // every reduced degree the schedule may need must exist with the same tile
        const int ty = p.ndim == 3 ? inst.tile_y : 0;
        bool ok = true;
        for (int d = 1; d < inst.bT && ok; ++d)
            ok = find_instance(p, d, inst.vec, direct, inst.tile_x_loaded, inst.threads, ty) != nullptr ||
                 find_instance(p, d, inst.vec, direct, inst.tile_x_loaded, 0, ty) != nullptr;
        if (!ok) continue;
        std::vector<int64_t> hs;
        if (hint && hint->h) {
            hs.push_back(hint->h);
        } else {
            SweepGeom g{};
            if (sweep_geometry(p, inst, dm, inst.bT, Iout, 0, dm.E[0], p.rad, dm.E[0] - p.rad, g) != AN5D_OK) continue;
            int64_t nt = 1;
            for (int i = 0; i < p.ndim - 1; ++i) nt *= g.ntiles[i];
            const int64_t conc = resident_units(inst);
            // stream-block lengths giving 1..32 units per resident block, and a few fixed lengths
            for (int w : {1, 2, 4, 8, 16, 32}) {
                const int64_t nsb = std::max<int64_t>(1, (w * conc) / std::max<int64_t>(1, nt));
                hs.push_back(std::max<int64_t>(1, cdiv(Iout, nsb)));
            }
            for (int64_t hh : {64, 128, 256, 512}) hs.push_back(std::min<int64_t>(hh, Iout));
            hs.push_back(Iout);
        }
        for (int64_t h : hs) {
            const double t = model_time(p, inst, dm, inst.bT, h, di, nullptr);
            if (t >= 1e29) continue;
            an5d_config c{};
            c.bT = inst.bT;
            c.vec = inst.vec;
            c.h = h;
            c.n_thr = inst.threads;
            {   // logical tile b_S = compute region + 2 b_T rad (names the layout, inst_matches)
                SweepGeom g{};
                sweep_geometry(p, inst, dm, inst.bT, h, 0, dm.E[0], p.rad, dm.E[0] - p.rad, g);
                for (int i = 0; i < p.ndim - 1; ++i) c.bS[i] = g.C[i] + 2 * inst.bT * p.rad;
            }
            c.direct = direct;
            out.emplace_back(t, c);
        }
    }
    std::stable_sort(out.begin(), out.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    return out;
}

an5d_status choose_config(const Plan& p, const Dims& dm, int64_t T, const an5d_config* hint, an5d_config& out) {
    const auto r = rank_configs(p, dm, T, hint);
    if (r.empty())
        return fail(AN5D_ERR_UNSUPPORTED, "no feasible kernel instance for ndim=%d rad=%d shape=%d dtype=%d",
                    p.ndim, p.rad, p.shape, p.dtype);
    out = r.front().second;
    return AN5D_OK;
}

// ---------------------------------------------------------------------------------------------
// Copy kernels (ring copy: O(surface); whole-array copy for T == 0 / trailing copy)
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void ring_copy_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t nrows, int64_t Ey,
                                 int64_t Ex, int64_t pz, int64_t py, int R, int64_t g_off, int64_t gE0,
                                 int is3d) {
    for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
        int64_t z = 0, y = row;
        if (is3d) { z = row / Ey; y = row % Ey; }
        const int64_t gouter = (is3d ? z : y) + g_off;
        bool full = gouter < R || gouter >= gE0 - R;
        if (is3d) full = full || y < R || y >= Ey - R;
        const int64_t off = is3d ? z * pz + y * py : y * py;
        if (full) {
            for (int64_t x = threadIdx.x; x < Ex; x += blockDim.x) dst[off + x] = src[off + x];
        } else {
            for (int64_t x = threadIdx.x; x < 2 * R; x += blockDim.x) {
                const int64_t xx = x < R ? x : Ex - 2 * R + x;
                dst[off + xx] = src[off + xx];
            }
        }
    }
}

template <typename T>
__global__ void copy_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t nrows, int64_t Ey,
                            int64_t Ex, int64_t pz, int64_t py, int is3d) {
    for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
        int64_t off = row * py;
        if (is3d) off = (row / Ey) * pz + (row % Ey) * py;
        for (int64_t x = threadIdx.x; x < Ex; x += blockDim.x) dst[off + x] = src[off + x];
    }
}

an5d_status launch_copy(Plan& p, const void* src, void* dst, const Dims& dm, bool ring_only, int64_t g_off,
                        int64_t gE0, cudaStream_t st) {
    const bool is3d = p.ndim == 3;
    const int64_t Ey = is3d ? dm.E[1] : dm.E[0];
    const int64_t Ex = dm.E[p.ndim - 1];
    const int64_t nrows = is3d ? dm.E[0] * dm.E[1] : dm.E[0];
    const int64_t pz = is3d ? dm.pitch[0] : 0;
    const int64_t py = is3d ? dm.pitch[1] : dm.pitch[0];
    const unsigned grid = (unsigned)std::min<int64_t>(nrows, 148 * 32);
    const int thr = ring_only ? 128 : 256;
    for (int f = 0; f < p.nf; ++f) {   // every field of a system (one for a plain stencil)
    src = static_cast<const char*>(src) + (f ? dm.fstride * (int64_t)p.elem : 0);
    dst = static_cast<char*>(dst) + (f ? dm.fstride * (int64_t)p.elem : 0);
    if (p.dtype == AN5D_F32) {
        if (ring_only)
            ring_copy_kernel<float><<<grid, thr, 0, st>>>((const float*)src, (float*)dst, nrows, Ey, Ex, pz, py,
                                                          p.rad, g_off, gE0, is3d);
        else
            copy_kernel<float><<<grid, thr, 0, st>>>((const float*)src, (float*)dst, nrows, Ey, Ex, pz, py, is3d);
    } else {
        if (ring_only)
            ring_copy_kernel<double><<<grid, thr, 0, st>>>((const double*)src, (double*)dst, nrows, Ey, Ex, pz,
                                                           py, p.rad, g_off, gE0, is3d);
        else
            copy_kernel<double><<<grid, thr, 0, st>>>((const double*)src, (double*)dst, nrows, Ey, Ex, pz, py,
                                                      is3d);
    }
    p.launches++;
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? AN5D_OK : cuda_fail(e, "copy kernel launch");
}

// Per-device plan state: the dynamic-scheduling counter pairs (zeroed) and the run-table cache.
an5d_status ensure_streams(Plan& p) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (p.ctr && p.device == dev) return AN5D_OK;
    if (p.ctr) cudaFree(p.ctr);
    for (auto& kv : p.runs) cudaFree(kv.second.first);
    p.runs.clear();
    // counter pairs + the scratch slots of the 2D kernels' no-op lane atomics (kScratch2D)
    const size_t n = 2 * kCtrRing + kScratch2D;
    if ((e = cudaMalloc(&p.ctr, sizeof(unsigned long long) * n)) != cudaSuccess) return cuda_fail(e, "counter");
    if ((e = cudaMemset(p.ctr, 0, sizeof(unsigned long long) * n)) != cudaSuccess) return cuda_fail(e, "counter");
    p.device = dev;
    return AN5D_OK;
}

// The TMA descriptor of a 3D sweep's input: the local array as a tensor {x, y, z} whose origin is
// moved back to the 16-byte boundary before x = 0 (TMA needs a 16-byte aligned base; the C ABI
// guarantees (base + rad*elem) % 16 == 0, so that boundary lies at most 12 bytes before the array
// inside the same allocation).  Box = one staged tile plane {kTX, kTY, 1}; out-of-bound parts
// (y < 0, y >= E_y, z outside the local array, x past the row end) are zero-filled by the TMA unit.
an5d_status encode_tmap_3d(const Plan& p, const Instance& inst, const void* src, const Dims& dm, CUtensorMap& tm,
                           int& x_off) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !f) {
            cudaGetLastError();
            return fail(AN5D_ERR_CUDA, "cuTensorMapEncodeTiled entry point not available");
        }
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    const uintptr_t base = reinterpret_cast<uintptr_t>(src);
    const uintptr_t aligned = base & ~uintptr_t(15);
    x_off = (int)((base - aligned) / p.elem);
    const cuuint64_t dims[3] = {(cuuint64_t)(dm.E[2] + x_off), (cuuint64_t)dm.E[1], (cuuint64_t)dm.E[0]};
    const cuuint64_t strides[2] = {(cuuint64_t)(dm.pitch[1] * p.elem), (cuuint64_t)(dm.pitch[0] * p.elem)};
    // one block's plane: a cluster layout's blocks each load their own tile_y / cluster rows
    // (a cluster layout's block also stages rad pad rows above and below: kernel3d.cuh kBoxRows)
    const int cl = std::max(1, inst.cluster);
    // (XPAIR: the box starts 2 cells before the window and is 4 cells wider, kernel3d.cuh kTXL)
    const cuuint32_t box[3] = {(cuuint32_t)(inst.tile_x_loaded + (inst.xpair ? 4 : 0)),
                               (cuuint32_t)(inst.tile_y / cl + (cl > 1 ? 2 * p.rad : 0)), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&tm, p.elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                        reinterpret_cast<void*>(aligned), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(AN5D_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return AN5D_OK;
}

// One sweep: one persistent launch (2D) or one block per run-table unit (3D), on the caller's stream.
// Peer-store fields of a sweep's argument block (fused halo exchange): element shifts from the
// per-plane strides.  Planes [out_lo, out_lo + n0) also go to the lower neighbour, [out_hi - n1,
// out_hi) to the upper one.
template <typename Args>
void set_peers(Args& a, const an5d_peer_store* ps, int64_t plane_stride, int64_t out_lo, int64_t out_hi) {
    a.peer_lo = a.peer_hi = nullptr;
    a.send_lo_end = out_lo;
    a.send_hi_begin = out_hi;
    if (!ps) return;
    if (ps->peer_dst[0] && ps->send_planes[0] > 0) {
        a.peer_lo = ps->peer_dst[0];
        a.peer_lo_shift = ps->peer_plane_shift[0] * plane_stride;
        a.send_lo_end = out_lo + ps->send_planes[0];
    }
    if (ps->peer_dst[1] && ps->send_planes[1] > 0) {
        a.peer_hi = ps->peer_dst[1];
        a.peer_hi_shift = ps->peer_plane_shift[1] * plane_stride;
        a.send_hi_begin = out_hi - ps->send_planes[1];
    }
}

// dry = true: everything up to the launch (geometry, run-table upload), no launch -- lets a caller
// upload the run tables of all its sweeps before it enqueues stream waits (an5d_run_slab).
an5d_status launch_sweep(Plan& p, const void* src, void* dst, const Dims& dm, int d, const an5d_config& cfg,
                         int64_t g_off, int64_t gE0, int64_t out_lo, int64_t out_hi, int32_t* wc,
                         const an5d_peer_store* peers, bool dry,
                         cudaStream_t st) {
    const Instance* inst = find_instance(p, d, cfg);
    if (!inst) return fail(AN5D_ERR_UNSUPPORTED, "no kernel instance for degree %d vec %d", d, cfg.vec);
    SweepGeom g{};
    an5d_status s = sweep_geometry(p, *inst, dm, d, cfg.h, g_off, gE0, out_lo, out_hi, g);
    if (s != AN5D_OK) return s;
    cudaError_t e;
    if (p.ndim == 2) {
        // one persistent launch over every (tile, stream block) unit, interior and edge alike
        Sweep2DArgs a{};
        a.src = src; a.dst = dst; a.pitch = dm.pitch[0];
        a.Ey = dm.E[0]; a.g_off = g_off; a.gEy = gE0; a.out_lo = out_lo; a.out_hi = out_hi;
        a.h = g.h; a.n_units = g.n_units; a.n_sb = g.n_sb;
        a.ctr = p.ctr + 2 * (p.ctr_seq++ % kCtrRing);
        a.scratch = p.ctr + 2 * kCtrRing;
        a.wc = wc; a.Ex = (int)dm.E[1]; a.C = g.C[0]; a.H = g.halo[0]; a.n_tiles_x = (int)g.ntiles[0];
        a.fstride = dm.fstride;
        set_peers(a, peers, dm.pitch[0], out_lo, out_hi);
        const int64_t cap = (int64_t)resident_blocks(*inst) * dev_info().n_sm;
        const int64_t blocks = std::min<int64_t>(g.n_units, cap);
        const double frac = run_frac();
        if (frac > 0) {
            const int64_t W = run_warps(blocks);
            const std::vector<int64_t> key = {d, g.ntiles[0], g.n_sb, g.sb_lo, g.sb_hi, W, (int64_t)(frac * 1e6)};
            auto it = p.runs.find(key);
            if (it == p.runs.end() && p.runs.size() >= kRunCache) {
                // bounded cache: a plan run over many geometries drops its tables (device-synchronous
                // free; the stream order of earlier launches that read them is respected)
                cudaDeviceSynchronize();
                for (auto& kv : p.runs) cudaFree(kv.second.first);
                p.runs.clear();
                it = p.runs.end();
            }
            if (it == p.runs.end()) {
                const std::vector<int4> tab = build_runs_2d(g, W, frac);
                int4* dtab = nullptr;
                if ((e = cudaMalloc(&dtab, sizeof(int4) * tab.size())) != cudaSuccess) return cuda_fail(e, "run table");
                if ((e = cudaMemcpy(dtab, tab.data(), sizeof(int4) * tab.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
                    return cuda_fail(e, "run table upload");
                it = p.runs.emplace(key, std::make_pair(dtab, (int64_t)tab.size())).first;
            }
            a.runs = it->second.first;
            a.n_units = it->second.second;
        }
        if (dry) return AN5D_OK;
        // AN5D_UNIT_PROFILE=path: debug-only per-unit timing dump (synchronises; never in benches)
        const char* prof_path = getenv("AN5D_UNIT_PROFILE");
        if (prof_path && !wc) cudaMalloc(&a.unit_ns, sizeof(long long) * 3 * a.n_units);
        if ((e = inst->launch2d(a, p.coeffs_dev_t.data(), blocks, false, st)) != cudaSuccess)
            return cuda_fail(e, "sweep launch");
        p.launches++;
        if (a.unit_ns) {
            std::vector<long long> h(3 * a.n_units);
            cudaStreamSynchronize(st);
            cudaMemcpy(h.data(), a.unit_ns, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
            cudaFree(a.unit_ns);
            if (FILE* f = fopen(prof_path, "a")) {
                fprintf(f, "# sweep degree %d n_units %lld ntx %lld h %lld blocks %lld\n", d, (long long)a.n_units,
                        (long long)g.ntiles[0], (long long)g.h, (long long)blocks);
                for (int64_t u = 0; u < a.n_units; ++u)
                    fprintf(f, "%lld %lld %lld %lld\n", (long long)u, h[3 * u], h[3 * u + 1], h[3 * u + 2]);
                fclose(f);
            }
        }
        return AN5D_OK;
    } else {
        // one block per (tile, stream block) unit; edge units are numbered first
        Sweep3DArgs a{};
        a.src = src; a.dst = dst; a.pz = dm.pitch[0]; a.py = dm.pitch[1];
        a.Ez = dm.E[0]; a.g_off = g_off; a.gEz = gE0; a.out_lo = out_lo; a.out_hi = out_hi;
        a.h = g.h; a.n_sb = g.n_sb; a.n_units = g.n_units; a.wc = wc;
        set_peers(a, peers, dm.pitch[0], out_lo, out_hi);
        const double frac = run_frac();
        if (frac > 0) {
            const int64_t W = run_warps(resident_units(*inst));
            const std::vector<int64_t> key = {3, d, g.ntiles[0], g.ntiles[1], g.n_sb, g.sb_lo, g.sb_hi, W,
                                              (int64_t)(frac * 1e6)};
            auto it = p.runs.find(key);
            if (it == p.runs.end() && p.runs.size() >= kRunCache) {
                // bounded cache: a plan run over many geometries drops its tables (device-synchronous
                // free; the stream order of earlier launches that read them is respected)
                cudaDeviceSynchronize();
                for (auto& kv : p.runs) cudaFree(kv.second.first);
                p.runs.clear();
                it = p.runs.end();
            }
            if (it == p.runs.end()) {
                const std::vector<int4> tab = build_runs_3d(g, W, frac);
                int4* dtab = nullptr;
                if ((e = cudaMalloc(&dtab, sizeof(int4) * tab.size())) != cudaSuccess) return cuda_fail(e, "run table");
                if ((e = cudaMemcpy(dtab, tab.data(), sizeof(int4) * tab.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
                    return cuda_fail(e, "run table upload");
                it = p.runs.emplace(key, std::make_pair(dtab, (int64_t)tab.size())).first;
            }
            a.runs = it->second.first;
            a.n_units = it->second.second;
        }
        if (dry) return AN5D_OK;
        a.Ey = (int)dm.E[1]; a.Ex = (int)dm.E[2];
        a.Cy = g.C[0]; a.Cx = g.C[1]; a.Hy = g.halo[0]; a.Hx = g.halo[1];
        a.nty = (int)g.ntiles[0]; a.ntx = (int)g.ntiles[1];
        CUtensorMap tm;
        if ((s = encode_tmap_3d(p, *inst, src, dm, tm, a.x_off)) != AN5D_OK) return s;
        if ((e = inst->launch3d(a, p.coeffs_dev_t.data(), tm, a.n_units, st)) != cudaSuccess)
            return cuda_fail(e, "sweep launch");
        p.launches++;
    }
    return AN5D_OK;
}

an5d_status read_dims(const Plan& p, const int64_t* extents, const int64_t* pitches, Dims& dm) {
    if (!extents) return fail(AN5D_ERR_INVALID_ARGUMENT, "extents is NULL");
    if (p.nf > 1 && pitches) {   // systems: pitches = {field stride, the usual ndim-1 pitches}
        dm.fstride = pitches[0];
        pitches += 1;
    }
    for (int i = 0; i < p.ndim; ++i) {
        dm.E[i] = extents[i];
        if (dm.E[i] < 2 * p.rad + 1)
            return fail(AN5D_ERR_SHAPE_MISMATCH, "extent[%d]=%lld < 2*rad+1 (no interior cell)", i,
                        (long long)dm.E[i]);
        if (dm.E[i] > (1LL << 30) && i > 0)
            return fail(AN5D_ERR_UNSUPPORTED, "blocked extent[%d] too large", i);
    }
    if (p.ndim == 2) {
        dm.pitch[0] = pitches ? pitches[0] : dm.E[1];
        if (dm.pitch[0] < dm.E[1]) return fail(AN5D_ERR_SHAPE_MISMATCH, "row pitch < x extent");
        if (p.nf > 1 && !dm.fstride) dm.fstride = dm.E[0] * dm.pitch[0];   // NULL pitches: dense fields
        if (p.nf > 1 && dm.fstride < dm.E[0] * dm.pitch[0])
            return fail(AN5D_ERR_SHAPE_MISMATCH, "field stride < rows * pitch (fields overlap)");
    } else {
        dm.pitch[1] = pitches ? pitches[1] : dm.E[2];
        dm.pitch[0] = pitches ? pitches[0] : dm.E[1] * dm.pitch[1];
        if (dm.pitch[1] < dm.E[2]) return fail(AN5D_ERR_SHAPE_MISMATCH, "row pitch < x extent");
        if (dm.pitch[0] < dm.E[1] * dm.pitch[1]) return fail(AN5D_ERR_SHAPE_MISMATCH, "plane pitch < rows*pitch");
    }
    return AN5D_OK;
}

an5d_status check_alignment(const Plan& p, const void* ptr, const Dims& dm, const char* name) {
    if (!ptr) return fail(AN5D_ERR_INVALID_ARGUMENT, "%s is NULL", name);
    const uintptr_t a = reinterpret_cast<uintptr_t>(ptr) + (uintptr_t)p.rad * p.elem;
    if (a % 16) return fail(AN5D_ERR_UNSUPPORTED, "%s: element x=rad of row 0 is not 16-byte aligned", name);
    for (int i = 0; i < p.ndim - 1; ++i)
        if ((dm.pitch[i] * (int64_t)p.elem) % 16)
            return fail(AN5D_ERR_UNSUPPORTED, "%s: pitch[%d]*elem_size not a multiple of 16 bytes", name, i);
    if ((dm.fstride * (int64_t)p.elem) % 16)
        return fail(AN5D_ERR_UNSUPPORTED, "%s: field stride*elem_size not a multiple of 16 bytes", name);
    return AN5D_OK;
}

an5d_status resolve_config(Plan& p, const Dims& dm, int64_t T, const an5d_config* cfg, an5d_config& c) {
    an5d_config hint{};
    if (cfg) hint = *cfg;
    if (p.shape == AN5D_GRADIENT) hint.direct = 1;   // non-associative: direct gather only
    if (const char* f = getenv("AN5D_FORCE_CFG")) {  // "bT,vec,h" benchmarking override
        int bt = 0, v = 0;
        long long h = 0;
        if (sscanf(f, "%d,%d,%lld", &bt, &v, &h) >= 1) {
            if (bt) hint.bT = bt;
            if (v) hint.vec = v;
            if (h) hint.h = h;
        }
    }
    if (hint.bT < 0 || hint.vec < 0 || hint.h < 0 || hint.n_thr < 0 || hint.bS[0] < 0 || hint.bS[1] < 0)
        return fail(AN5D_ERR_INVALID_ARGUMENT, "negative config field");
    if (hint.direct != 0 && hint.direct != 1) return fail(AN5D_ERR_INVALID_ARGUMENT, "direct must be 0 or 1");
    if (hint.bT && hint.vec && hint.h) {
        c = hint;
    } else {
        an5d_status s = choose_config(p, dm, T, &hint, c);
        if (s != AN5D_OK) return s;
    }
    if (c.direct && p.ndim != 2)
        return fail(AN5D_ERR_UNSUPPORTED, "direct (non-associative) variant is 2D only");
    const Instance* inst = find_instance(p, c.bT, c);
    if (!inst)
        return fail(AN5D_ERR_UNSUPPORTED,
                    "no kernel instance for ndim=%d rad=%d shape=%d dtype=%d bT=%d vec=%d bS=(%d,%d) n_thr=%d", p.ndim,
                    p.rad, p.shape, p.dtype, c.bT, c.vec, c.bS[0], c.bS[1], c.n_thr);
    c.n_thr = inst->threads;
    for (int d = 1; d < c.bT; ++d)
        if (!find_instance(p, d, c))
            return fail(AN5D_ERR_UNSUPPORTED, "no reduced-degree instance d=%d for vec %d", d, c.vec);
    // logical tile b_S reported back
    SweepGeom g{};
    an5d_status s = sweep_geometry(p, *inst, dm, c.bT, c.h ? c.h : dm.E[0], 0, dm.E[0], p.rad, dm.E[0] - p.rad, g);
    if (s != AN5D_OK) return s;
    const int nb = p.ndim - 1;
    for (int i = 0; i < 2; ++i) {
        const int want = i < nb ? g.C[i] + 2 * c.bT * p.rad : 0;
        if (cfg && cfg->bS[i] && cfg->bS[i] != want)
            return fail(AN5D_ERR_UNSUPPORTED, "bS[%d]=%d not available: instance vec=%d gives b_S=%d", i, cfg->bS[i],
                        c.vec, want);
        c.bS[i] = want;
    }
    if (!c.h) c.h = dm.E[0] - 2 * p.rad;
    return AN5D_OK;
}

}  // namespace
// Coefficient table in the run's dtype, with the j-stencil divisor folded in (R-8:
// the paper's fast-math build turns "/c_0" into a multiply; here it costs
// nothing at all because 1/c_0 is folded into the taps).
//   divisor == 1: every coefficient rounded once to nearest (the oracle uses the same values).
//   divisor != 1: each folded tap is one of the two dtype neighbours of c_d / c_0, chosen so that
//   the taps' exact sum is as close as possible to sum_d c_d / c_0 (compensated rounding).  Plain
//   rounding to nearest leaves a systematic bias (sum of taps = 1 + eps) that a T-step run
//   amplifies T-fold: j2d9pt fp32, T = 1000 drifted 1.1e-5 from the oracle (reading R-8b).
template <typename T>
std::vector<T> fold_coefficients(const double* c, size_t n, double divisor) {
    std::vector<T> out(n);
    if (divisor == 1.0) {
        for (size_t k = 0; k < n; ++k) out[k] = (T)c[k];
        return out;
    }
    std::vector<long double> q(n);
    long double target = 0, sum = 0;
    for (size_t k = 0; k < n; ++k) {
        q[k] = (long double)c[k] / (long double)divisor;
        target += q[k];
        out[k] = (T)q[k];
        sum += (long double)out[k];
    }
    std::vector<char> flipped(n, 0);
    for (size_t it = 0; it < n; ++it) {
        const long double err = sum - target;
        size_t best = n;
        long double best_err = fabsl(err);
        T best_v = 0;
        for (size_t k = 0; k < n; ++k) {
            if (flipped[k] || q[k] == (long double)out[k]) continue;
            // the other neighbour of q[k]
            const T other = (long double)out[k] < q[k] ? std::nextafter(out[k], (T)INFINITY)
                                                       : std::nextafter(out[k], (T)-INFINITY);
            const long double e2 = err - (long double)out[k] + (long double)other;
            if (fabsl(e2) < best_err) {
                best_err = fabsl(e2);
                best = k;
                best_v = other;
            }
        }
        if (best == n) break;
        sum += (long double)best_v - (long double)out[best];
        out[best] = best_v;
        flipped[best] = 1;
    }
    return out;
}

}  // namespace an5d

using namespace an5d;

namespace {
typedef CUresult (*StreamValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*AddressRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
template <typename F>
F driver_fn(const char* name) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return reinterpret_cast<F>(f);
}
}  // namespace

// =============================================================================================
// NCCL slab mode (an5d_set_comm).  NCCL is loaded at run time so the
// library never pins a second NCCL next to the one the process (torch) already has.
// =============================================================================================
namespace {
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = nullptr;
    if (const char* e = getenv("AN5D_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);   // already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { api.why = std::string("cannot load libnccl.so.2: ") + dlerror(); return api; }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
             api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    return api;
}

an5d_status nccl_fail(ncclResult_t r, const char* what) {
    return fail(AN5D_ERR_NCCL, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
}

// One rank's T-step run of its slab with the NCCL exchange (mirrors slab.py run_distributed):
// per sweep the boundary output planes first, then the d_next rad outermost owned planes are
// sent to / received from the neighbours on the plan's comm stream while the interior planes are
// computed on `st`; the next sweep waits for the exchange.
an5d_status run_comm(Plan& p, void* grid_in, void* grid_out, const Dims& dm, int64_t T, const an5d_config& c,
                     cudaStream_t st) {
    const NcclApi& api = nccl();
    std::vector<int> deg;
    bool tc = false;
    make_schedule(T, c.bT, deg, tc);
    const int R = p.rad;
    const bool lower = p.rank > 0, upper = p.rank < p.nranks - 1;
    const int64_t E0 = dm.E[0];
    const int64_t out_lo = lower ? p.ghost : std::max<int64_t>(0, R - p.outer_offset);
    const int64_t out_hi = upper ? E0 - p.ghost : std::min<int64_t>(E0, p.gE0 - R - p.outer_offset);
    if ((lower || upper) && p.ghost < c.bT * R)
        return fail(AN5D_ERR_UNSUPPORTED, "ghost_planes %d < b_T * rad = %d", p.ghost, c.bT * R);
    if (out_hi <= out_lo) return fail(AN5D_ERR_SHAPE_MISMATCH, "slab owns no plane");
    for (int d : deg) {   // validate every sweep before the first launch
        const Instance* inst = find_instance(p, d, c);
        SweepGeom g{};
        an5d_status s = sweep_geometry(p, *inst, dm, d, c.h, p.outer_offset, p.gE0, out_lo, out_hi, g);
        if (s != AN5D_OK) return s;
    }
    an5d_status s = launch_copy(p, grid_in, grid_out, dm, true, p.outer_offset, p.gE0, st);
    if (s != AN5D_OK) return s;
    const size_t plane_bytes = (size_t)dm.pitch[0] * p.elem;
    void* bufs[2] = {grid_in, grid_out};
    bool pending = false;
    cudaError_t e;
    for (size_t i = 0; i < deg.size(); ++i) {
        const void* src = bufs[i % 2];
        char* dst = static_cast<char*>(bufs[(i + 1) % 2]);
        const int d = deg[i], nd = i + 1 < deg.size() ? deg[i + 1] : 0;
        const int64_t g = (int64_t)nd * R, hb = std::max<int64_t>(g, c.h);
        int64_t blo = (lower && g) ? out_lo + hb : out_lo, bhi = (upper && g) ? out_hi - hb : out_hi;
        std::vector<std::pair<int64_t, int64_t>> boundary, interior;
        if (blo >= bhi) {
            boundary.emplace_back(out_lo, out_hi);
        } else {
            if (blo > out_lo) boundary.emplace_back(out_lo, blo);
            if (out_hi > bhi) boundary.emplace_back(bhi, out_hi);
            interior.emplace_back(blo, bhi);
        }
        if (pending && (e = cudaStreamWaitEvent(st, p.ev_xchg, 0)) != cudaSuccess) return cuda_fail(e, "wait exchange");
        pending = false;
        for (auto& r : boundary)
            if ((s = launch_sweep(p, src, dst, dm, d, c, p.outer_offset, p.gE0, r.first, r.second, nullptr, nullptr,
                                  false, st)) != AN5D_OK)
                return s;
        if (g && (lower || upper)) {
            if ((e = cudaEventRecord(p.ev_bnd, st)) != cudaSuccess) return cuda_fail(e, "event");
            if ((e = cudaStreamWaitEvent(p.comm_stream, p.ev_bnd, 0)) != cudaSuccess) return cuda_fail(e, "wait");
            ncclResult_t r = api.GroupStart();
            if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
            const size_t n = (size_t)g * plane_bytes;
            if (lower) {
                if ((r = api.Send(dst + out_lo * plane_bytes, n, ncclUint8, p.rank - 1, p.comm, p.comm_stream)) != ncclSuccess)
                    return nccl_fail(r, "ncclSend");
                if ((r = api.Recv(dst + (out_lo - g) * plane_bytes, n, ncclUint8, p.rank - 1, p.comm, p.comm_stream)) !=
                    ncclSuccess)
                    return nccl_fail(r, "ncclRecv");
            }
            if (upper) {
                if ((r = api.Send(dst + (out_hi - g) * plane_bytes, n, ncclUint8, p.rank + 1, p.comm, p.comm_stream)) !=
                    ncclSuccess)
                    return nccl_fail(r, "ncclSend");
                if ((r = api.Recv(dst + out_hi * plane_bytes, n, ncclUint8, p.rank + 1, p.comm, p.comm_stream)) != ncclSuccess)
                    return nccl_fail(r, "ncclRecv");
            }
            if ((r = api.GroupEnd()) != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
            if ((e = cudaEventRecord(p.ev_xchg, p.comm_stream)) != cudaSuccess) return cuda_fail(e, "event");
            pending = true;
        }
        for (auto& r : interior)
            if ((s = launch_sweep(p, src, dst, dm, d, c, p.outer_offset, p.gE0, r.first, r.second, nullptr, nullptr,
                                  false, st)) != AN5D_OK)
                return s;
    }
    if (pending && (e = cudaStreamWaitEvent(st, p.ev_xchg, 0)) != cudaSuccess) return cuda_fail(e, "wait exchange");
    if (tc) return launch_copy(p, grid_in, grid_out, dm, false, 0, E0, st);   // b_T = 1, even count
    return AN5D_OK;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

const char* an5d_last_error(void) { return g_err.c_str(); }
const char* an5d_version(void) { return "an5d-b200 0.1 (sm_100a)"; }

an5d_status an5d_create(int ndim, int radius, an5d_shape shape, const double* coeffs, size_t n_coeffs,
                        double divisor, an5d_dtype dtype, an5d_plan** out) {
    try {
        if (!out) return fail(AN5D_ERR_INVALID_ARGUMENT, "out is NULL");
        *out = nullptr;
        if (ndim != 2 && ndim != 3) return fail(AN5D_ERR_INVALID_ARGUMENT, "ndim must be 2 or 3");
        if (radius < 1 || radius > 4) return fail(AN5D_ERR_INVALID_ARGUMENT, "radius must be 1..4");
        if (shape != AN5D_STAR && shape != AN5D_BOX && shape != AN5D_GRADIENT)
            return fail(AN5D_ERR_INVALID_ARGUMENT, "bad shape");
        if (shape == AN5D_GRADIENT && (ndim != 2 || radius != 1))
            return fail(AN5D_ERR_UNSUPPORTED, "gradient2d is ndim 2, radius 1 (Table 2 P:698-699)");
        // gradient2d: c_0 + (sum of squares) must stay a normal number for the kernel's
        // branch-free correctly rounded 1/sqrt (kernel2d.cuh rn_rsqrt_div)
        if (shape == AN5D_GRADIENT && !(divisor >= (dtype == AN5D_F32 ? 1.1754943508222875e-38 : 2.2250738585072014e-308)))
            return fail(AN5D_ERR_UNSUPPORTED, "gradient2d needs c_0 >= the dtype's smallest normal number");
        if (dtype != AN5D_F32 && dtype != AN5D_F64) return fail(AN5D_ERR_INVALID_ARGUMENT, "bad dtype");
        if (!coeffs) return fail(AN5D_ERR_INVALID_ARGUMENT, "coeffs is NULL");
        if (!(divisor != 0.0) || !std::isfinite(divisor)) return fail(AN5D_ERR_INVALID_ARGUMENT, "bad divisor");
        const int w = 2 * radius + 1;
        const size_t n = ndim == 2 ? (size_t)w * w : (size_t)w * w * w;
        if (n_coeffs != n)
            return fail(AN5D_ERR_SHAPE_MISMATCH, "expected %zu coefficients ((2r+1)^ndim), got %zu", n, n_coeffs);
        for (size_t k = 0; k < n; ++k) {
            int rem = (int)k, nz = 0;
            for (int i = 0; i < ndim; ++i) { nz += (rem % w) != radius; rem /= w; }
            if (!std::isfinite(coeffs[k])) return fail(AN5D_ERR_INVALID_ARGUMENT, "non-finite coefficient");
            if (shape == AN5D_STAR && nz > 1 && coeffs[k] != 0.0)
                return fail(AN5D_ERR_SHAPE_MISMATCH, "STAR table has non-zero off-axis entry %zu", k);
            if (shape == AN5D_GRADIENT && nz > 0 && coeffs[k] != 0.0)
                return fail(AN5D_ERR_SHAPE_MISMATCH, "GRADIENT table has non-zero off-centre entry %zu", k);
        }
        an5d_plan* p = new an5d_plan();
        p->ndim = ndim; p->rad = radius; p->shape = shape; p->dtype = dtype;
        p->elem = dtype == AN5D_F32 ? 4 : 8;
        p->divisor = divisor;
        p->coeffs_folded.resize(n);
        p->coeffs_dev_t.resize(n * p->elem);
        if (shape == AN5D_GRADIENT) {
            // gradient2d: the table rounded once (its centre is c) followed by c_0 = `divisor`,
            // rounded once; nothing is folded (the divisor is not a divisor here)
            p->coeffs_dev_t.resize((n + 1) * p->elem);
            for (size_t k = 0; k <= n; ++k) {
                const double v = k < n ? coeffs[k] : divisor;
                if (dtype == AN5D_F32) {
                    const float f = (float)v;
                    memcpy(p->coeffs_dev_t.data() + k * 4, &f, 4);
                    if (k < n) p->coeffs_folded[k] = f;
                } else {
                    memcpy(p->coeffs_dev_t.data() + k * 8, &v, 8);
                    if (k < n) p->coeffs_folded[k] = v;
                }
            }
        } else if (dtype == AN5D_F32) {
            const std::vector<float> f = fold_coefficients<float>(coeffs, n, divisor);
            memcpy(p->coeffs_dev_t.data(), f.data(), n * 4);
            for (size_t k = 0; k < n; ++k) p->coeffs_folded[k] = f[k];
        } else {
            const std::vector<double> f = fold_coefficients<double>(coeffs, n, divisor);
            memcpy(p->coeffs_dev_t.data(), f.data(), n * 8);
            for (size_t k = 0; k < n; ++k) p->coeffs_folded[k] = f[k];
        }
        *out = p;
        return AN5D_OK;
    } catch (const std::bad_alloc&) {
        return fail(AN5D_ERR_OUT_OF_MEMORY, "host allocation failed");
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

an5d_status an5d_create_system(int ndim, int radius, an5d_shape shape, int n_fields, const double* coeffs,
                               size_t n_coeffs, an5d_dtype dtype, an5d_plan** out) {
    try {
        if (!out) return fail(AN5D_ERR_INVALID_ARGUMENT, "out is NULL");
        *out = nullptr;
        if (n_fields < 1 || n_fields > 8) return fail(AN5D_ERR_INVALID_ARGUMENT, "n_fields must be 1..8");
        if (shape != AN5D_STAR && shape != AN5D_BOX) return fail(AN5D_ERR_INVALID_ARGUMENT, "bad shape");
        if (ndim != 2 && ndim != 3) return fail(AN5D_ERR_INVALID_ARGUMENT, "ndim must be 2 or 3");
        if (radius < 1 || radius > 4) return fail(AN5D_ERR_INVALID_ARGUMENT, "radius must be 1..4");
        if (dtype != AN5D_F32 && dtype != AN5D_F64) return fail(AN5D_ERR_INVALID_ARGUMENT, "bad dtype");
        if (!coeffs) return fail(AN5D_ERR_INVALID_ARGUMENT, "coeffs is NULL");
        const int w = 2 * radius + 1;
        const size_t n = ndim == 2 ? (size_t)w * w : (size_t)w * w * w;
        const size_t nb = (size_t)n_fields * n_fields;
        if (n_coeffs != n * nb)
            return fail(AN5D_ERR_SHAPE_MISMATCH, "expected %zu coefficients (n_fields^2 (2r+1)^ndim), got %zu", n * nb,
                        n_coeffs);
        if (ndim != 2 && n_fields > 1) return fail(AN5D_ERR_UNSUPPORTED, "multi-field systems are 2D");
        an5d_plan* p = nullptr;
        an5d_status s = an5d_create(ndim, radius, shape, coeffs, n, 1.0, dtype, &p);   // validates block 0
        if (s != AN5D_OK) return s;
        p->nf = n_fields;
        p->coeffs_dev_t.resize(n * nb * p->elem);
        for (size_t k = 0; k < n * nb; ++k) {
            int rem = (int)(k % n), nz = 0;
            for (int i = 0; i < ndim; ++i) { nz += (rem % w) != radius; rem /= w; }
            if (!std::isfinite(coeffs[k]) || (shape == AN5D_STAR && nz > 1 && coeffs[k] != 0.0)) {
                an5d_destroy(p);
                return fail(AN5D_ERR_SHAPE_MISMATCH, "bad coefficient %zu (non-finite or STAR off-axis)", k);
            }
            if (dtype == AN5D_F32) {   // rounded once to the dtype (nothing to fold: no divisor)
                const float f = (float)coeffs[k];
                memcpy(p->coeffs_dev_t.data() + k * 4, &f, 4);
            } else {
                memcpy(p->coeffs_dev_t.data() + k * 8, &coeffs[k], 8);
            }
        }
        *out = p;
        return AN5D_OK;
    } catch (const std::bad_alloc&) {
        return fail(AN5D_ERR_OUT_OF_MEMORY, "host allocation failed");
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

an5d_status an5d_comm_unique_id(void* out128) {
    if (!out128) return fail(AN5D_ERR_INVALID_ARGUMENT, "out is NULL");
    const NcclApi& api = nccl();
    if (!api.ok) return fail(AN5D_ERR_NCCL, "%s", api.why.c_str());
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(out128, &id, sizeof(id));
    return AN5D_OK;
}

an5d_status an5d_set_comm(an5d_plan* p, const void* nccl_unique_id, int rank, int nranks, int64_t global_outer_extent,
                          int64_t outer_offset, int ghost_planes) {
    try {
        if (!p) return fail(AN5D_ERR_INVALID_ARGUMENT, "plan is NULL");
        if (p->comm) {   // detach the previous communicator (stream-ordered work must be done)
            if (p->comm_stream) cudaStreamSynchronize(p->comm_stream);
            nccl().CommDestroy(p->comm);
            p->comm = nullptr;
        }
        if (p->comm_stream) { cudaStreamDestroy(p->comm_stream); p->comm_stream = nullptr; }
        if (p->ev_bnd) { cudaEventDestroy(p->ev_bnd); p->ev_bnd = nullptr; }
        if (p->ev_xchg) { cudaEventDestroy(p->ev_xchg); p->ev_xchg = nullptr; }
        p->rank = 0; p->nranks = 1; p->ghost = 0; p->gE0 = 0; p->outer_offset = 0;
        if (!nccl_unique_id) return AN5D_OK;
        if (nranks < 1 || rank < 0 || rank >= nranks) return fail(AN5D_ERR_INVALID_ARGUMENT, "bad rank / nranks");
        if (ghost_planes < 0 || global_outer_extent < 2 * p->rad + 1 || outer_offset < 0)
            return fail(AN5D_ERR_INVALID_ARGUMENT, "bad ghost_planes / global_outer_extent / outer_offset");
        if (p->nf > 1) return fail(AN5D_ERR_UNSUPPORTED, "slab mode: single-field plans only");
        const NcclApi& api = nccl();
        if (!api.ok) return fail(AN5D_ERR_NCCL, "%s", api.why.c_str());
        ncclUniqueId id;
        memcpy(&id, nccl_unique_id, sizeof(id));
        ncclComm_t comm = nullptr;
        ncclResult_t r = api.CommInitRank(&comm, nranks, id, rank);
        if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
        cudaError_t e;
        if ((e = cudaStreamCreateWithFlags(&p->comm_stream, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&p->ev_bnd, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&p->ev_xchg, cudaEventDisableTiming)) != cudaSuccess) {
            api.CommDestroy(comm);
            return cuda_fail(e, "comm stream / events");
        }
        p->comm = comm;
        p->rank = rank; p->nranks = nranks; p->ghost = ghost_planes;
        p->gE0 = global_outer_extent; p->outer_offset = outer_offset;
        return AN5D_OK;
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

an5d_status an5d_destroy(an5d_plan* p) {
    if (!p) return AN5D_OK;
    an5d_set_comm(p, nullptr, 0, 1, 0, 0, 0);   // releases a communicator, if any
    if (p->ctr) cudaFree(p->ctr);
    for (auto& kv : p->runs) cudaFree(kv.second.first);
    delete p;
    return AN5D_OK;
}

int64_t an5d_last_launch_count(const an5d_plan* p) { return p ? p->launches : 0; }

an5d_status an5d_schedule(int64_t T, int bT, int* degrees, int64_t cap, int64_t* n_sweeps, int* trailing_copy) {
    try {
        if (T < 0 || bT < 1) return fail(AN5D_ERR_INVALID_ARGUMENT, "T < 0 or bT < 1");
        std::vector<int> deg;
        bool tc = false;
        make_schedule(T, bT, deg, tc);
        if (n_sweeps) *n_sweeps = (int64_t)deg.size();
        if (trailing_copy) *trailing_copy = tc ? 1 : 0;
        if (degrees)
            for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)deg.size()); ++i) degrees[i] = deg[i];
        return AN5D_OK;
    } catch (...) {
        return fail(AN5D_ERR_OUT_OF_MEMORY, "schedule");
    }
}

an5d_status an5d_plan_config(an5d_plan* p, const int64_t* extents, int64_t T, const an5d_config* hint,
                             an5d_config* out) {
    try {
        if (!p || !out) return fail(AN5D_ERR_INVALID_ARGUMENT, "NULL argument");
        Dims dm{};
        an5d_status s = read_dims(*p, extents, nullptr, dm);
        if (s != AN5D_OK) return s;
        return resolve_config(*p, dm, T, hint, *out);
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

// The paper's tuning procedure: rank every configuration with the model, run the top
// few on the GPU, keep the fastest.  Candidates are the best stream-block length of each of the
// top_k distinct (b_T, vec, layout) triples; each is timed over two sweeps (after one warm-up sweep) reading
// grid_in and writing grid_out.  Blocking: synchronises cuda_stream.
an5d_status an5d_tune(an5d_plan* p, const void* grid_in, void* grid_out, const int64_t* extents,
                      const int64_t* pitches, int64_t T, const an5d_config* hint, int top_k, an5d_config* out,
                      double* best_seconds_per_cell_step, void* stream) {
    try {
        if (!p || !out || !grid_in || !grid_out) return fail(AN5D_ERR_INVALID_ARGUMENT, "NULL argument");
        if (top_k < 1) return fail(AN5D_ERR_INVALID_ARGUMENT, "top_k < 1");
        if (grid_in == grid_out) return fail(AN5D_ERR_INVALID_ARGUMENT, "grid_in and grid_out must differ");
        Dims dm{};
        an5d_status s = read_dims(*p, extents, pitches, dm);
        if (s != AN5D_OK) return s;
        if ((s = check_alignment(*p, grid_in, dm, "grid_in")) != AN5D_OK) return s;
        if ((s = check_alignment(*p, grid_out, dm, "grid_out")) != AN5D_OK) return s;
        an5d_config h{};
        if (hint) h = *hint;
        if (h.bT < 0 || h.vec < 0 || h.h < 0 || (h.direct != 0 && h.direct != 1))
            return fail(AN5D_ERR_INVALID_ARGUMENT, "bad hint");
        const auto ranked = rank_configs(*p, dm, T, &h);
        // candidates: the top_k distinct (b_T, vec) pairs of the model's ranking, each with the
        // model's best configuration of EVERY kernel layout (threads x tile width) it has, plus
        // the best configuration of any layout still missing.  The model orders b_T well but the
        // layouts only roughly (measured on B200: the 2D level split ranks high in the model and
        // runs 8-20 % slower; the 512-thread fp64 3D layout runs 15-30 % faster), so every layout
        // is measured rather than ranked.
        auto layout_of = [&](const an5d_config& c) {
            const Instance* i = find_instance(*p, c.bT, c);
            return std::make_tuple(c.vec, c.n_thr, i ? i->tile_x_loaded : 0, i ? i->tile_y : 0);
        };
        std::vector<std::pair<int, int>> pairs;
        for (const auto& r : ranked) {
            const std::pair<int, int> bv(r.second.bT, r.second.vec);
            if (std::find(pairs.begin(), pairs.end(), bv) == pairs.end()) pairs.push_back(bv);
            if ((int)pairs.size() >= top_k) break;
        }
        std::vector<an5d_config> cand;
        auto add_if_new_layout = [&](const an5d_config& c, bool same_bT) {
            for (const auto& x : cand)
                if (layout_of(x) == layout_of(c) && (!same_bT || x.bT == c.bT)) return;
            cand.push_back(c);
        };
        for (const auto& r : ranked)
            if (std::find(pairs.begin(), pairs.end(), std::make_pair(r.second.bT, r.second.vec)) != pairs.end())
                add_if_new_layout(r.second, true);
        for (const auto& r : ranked) add_if_new_layout(r.second, false);
        if (cand.empty())
            return fail(AN5D_ERR_UNSUPPORTED, "no feasible kernel instance for ndim=%d rad=%d shape=%d dtype=%d",
                        p->ndim, p->rad, p->shape, p->dtype);
        if ((s = ensure_streams(*p)) != AN5D_OK) return s;
        cudaStream_t st = (cudaStream_t)stream;
        cudaEvent_t e0, e1;
        cudaError_t e;
        if ((e = cudaEventCreate(&e0)) != cudaSuccess) return cuda_fail(e, "event");
        if ((e = cudaEventCreate(&e1)) != cudaSuccess) { cudaEventDestroy(e0); return cuda_fail(e, "event"); }
        int64_t interior = 1;
        for (int i = 0; i < p->ndim; ++i) interior *= dm.E[i] - 2 * p->rad;
        double best = 1e300;
        an5d_config bc{};
        const int64_t launches0 = p->launches;
        // one warm-up sweep + two timed sweeps of a configuration: seconds per cell-step (1e300 if
        // it cannot run)
        // one warm-up sweep, then timed sweeps for >= 20 ms (at least 2, at most 96); every candidate
        // is timed in five passes (alternating forward / backward) and scored by its median pass: under
        // the 1 kW power cap the clocks drift by up to 10 % within a tune, which ordered short
        // single passes by the candidates' position rather than their speed (round-2 measurements)
        auto measure = [&](const an5d_config& c0, an5d_config& c) -> double {
            if (resolve_config(*p, dm, T, &c0, c) != AN5D_OK) return 1e300;
            auto sweep = [&]() {
                return launch_sweep(*p, grid_in, grid_out, dm, c.bT, c, 0, dm.E[0], p->rad, dm.E[0] - p->rad,
                                    nullptr, nullptr, false, st) == AN5D_OK;
            };
            bool ok = sweep();
            cudaEventRecord(e0, st);
            ok = ok && sweep();
            cudaEventRecord(e1, st);
            if (cudaEventSynchronize(e1) != cudaSuccess || !ok) {
                cudaGetLastError();
                return 1e300;
            }
            float ms1 = 0;
            cudaEventElapsedTime(&ms1, e0, e1);
            const int n = std::max(2, std::min(96, (int)std::ceil(20.0 / std::max(ms1, 1e-3f))));
            cudaEventRecord(e0, st);
            for (int r = 0; r < n && ok; ++r) ok = sweep();
            cudaEventRecord(e1, st);
            if (cudaEventSynchronize(e1) != cudaSuccess || !ok) {
                cudaGetLastError();
                return 1e300;
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            return ms * 1e-3 / n / ((double)interior * c.bT);
        };
        // bring the clocks up before the first candidate is timed (~50 ms of the model's pick)
        {
            an5d_config c{};
            if (resolve_config(*p, dm, T, &cand.front(), c) == AN5D_OK) {
                cudaEventRecord(e0, st);
                for (int r = 0; r < 64; ++r) {
                    launch_sweep(*p, grid_in, grid_out, dm, c.bT, c, 0, dm.E[0], p->rad, dm.E[0] - p->rad, nullptr,
                                 nullptr, false, st);
                    if (r == 0) {
                        cudaEventRecord(e1, st);
                        cudaEventSynchronize(e1);
                        float ms = 0;
                        cudaEventElapsedTime(&ms, e0, e1);
                        if (ms * 64 > 50.0f) r = 64 - std::max(1, (int)(50.0f / std::max(ms, 1e-3f)));
                    }
                }
                cudaStreamSynchronize(st);
                cudaGetLastError();
            }
        }
        const bool tlog = getenv("AN5D_TUNE_LOG") != nullptr;   // debug: every candidate's time
        // five passes (alternating forward / backward), each candidate scored by its median pass
        // (three passes still flipped star2d1r between b_T 7 and 8 -- 5 % apart -- from run to run
        // under the power cap, r02final/r02final2)
        constexpr int kPasses = 5;
        std::vector<std::vector<double>> times(cand.size());
        std::vector<double> score(cand.size(), 1e300);
        std::vector<an5d_config> resolved(cand.size());
        for (int pass = 0; pass < kPasses; ++pass)
            for (size_t j = 0; j < cand.size(); ++j) {
                const size_t q = (pass & 1) ? cand.size() - 1 - j : j;
                const double t = measure(cand[q], resolved[q]);
                times[q].push_back(t);
                if ((int)times[q].size() == kPasses) {
                    std::vector<double> v = times[q];
                    std::sort(v.begin(), v.end());
                    score[q] = v[kPasses / 2];
                }
                if (tlog)
                    fprintf(stderr, "an5d_tune: pass %d bT %d vec %d n_thr %d bS %d,%d h %lld -> %.4g ps/cell-step\n",
                            pass, cand[q].bT, cand[q].vec, cand[q].n_thr, cand[q].bS[0], cand[q].bS[1],
                            (long long)cand[q].h, t * 1e12);
            }
        for (size_t q = 0; q < cand.size(); ++q)
            if (score[q] < best) {
                best = score[q];
                bc = resolved[q];
            }
        // Final duel of the three best by median: interleaved rounds (each candidate timed for
        // >= 20 ms per round, the order rotated every round), summed.  Within a pass the clocks
        // drift under the power cap, and whichever candidate ran first measured up to 5 % faster
        // (AN5D_TUNE_LOG, r02p): the medians alone still flipped b_T 7 / 8 for star2d1r.
        {
            std::vector<size_t> order(cand.size());
            for (size_t q = 0; q < order.size(); ++q) order[q] = q;
            std::sort(order.begin(), order.end(), [&](size_t x, size_t y) { return score[x] < score[y]; });
            const size_t nd = std::min<size_t>(3, order.size());
            if (nd >= 2 && score[order[1]] < 1e299) {
                std::vector<double> sum(nd, 0.0);
                constexpr int kRounds = 6;
                for (int r = 0; r < kRounds; ++r)
                    for (size_t j = 0; j < nd; ++j) {
                        const size_t k = (j + (size_t)r) % nd;
                        an5d_config c{};
                        sum[k] += measure(cand[order[k]], c);
                    }
                size_t w = 0;
                for (size_t k = 1; k < nd; ++k)
                    if (sum[k] < sum[w]) w = k;
                if (tlog)
                    for (size_t k = 0; k < nd; ++k)
                        fprintf(stderr, "an5d_tune: duel bT %d vec %d n_thr %d h %lld -> %.4g ps/cell-step%s\n",
                                cand[order[k]].bT, cand[order[k]].vec, cand[order[k]].n_thr,
                                (long long)cand[order[k]].h, sum[k] / kRounds * 1e12, k == w ? " *" : "");
                bc = resolved[order[w]];
                best = sum[w] / kRounds;
            }
        }
        // stream-block length refinement around the model's pick for the winning (b_T, V) (the
        // model ranks h coarsely; measured on B200, star2d1r b_T 7: h 48 beats the model's 60 by 1.5 %)
        if (!h.h && best < 1e299) {
            const an5d_config base = bc;
            {   // re-time the winner so its neighbours are compared under the same clocks
                an5d_config c{};
                const double t = measure(base, c);
                if (t < 1e299) best = t;
            }
            for (double f : {0.5, 0.75, 1.5}) {
                an5d_config c0 = base, c{};
                c0.h = std::max<int64_t>(8, (int64_t)std::llround((double)base.h * f));
                if (c0.h == base.h) continue;
                const double t = measure(c0, c);
                if (tlog) fprintf(stderr, "an5d_tune: refine h %lld -> %.4g ps/cell-step\n", (long long)c0.h, t * 1e12);
                if (t < best) {
                    best = t;
                    bc = c;
                }
            }
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        p->launches = launches0;
        if (best >= 1e299) return fail(AN5D_ERR_CUDA, "no candidate configuration ran");
        *out = bc;
        if (best_seconds_per_cell_step) *best_seconds_per_cell_step = best;
        return AN5D_OK;
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

an5d_status an5d_describe(an5d_plan* p, const int64_t* extents, const an5d_config* cfg, an5d_geometry* out) {
    try {
        if (!p || !out || !cfg) return fail(AN5D_ERR_INVALID_ARGUMENT, "NULL argument");
        Dims dm{};
        an5d_status s = read_dims(*p, extents, nullptr, dm);
        if (s != AN5D_OK) return s;
        an5d_config c{};
        if ((s = resolve_config(*p, dm, 0, cfg, c)) != AN5D_OK) return s;
        const Instance* inst = find_instance(*p, c.bT, c);
        SweepGeom g{};
        if ((s = sweep_geometry(*p, *inst, dm, c.bT, c.h, 0, dm.E[0], p->rad, dm.E[0] - p->rad, g)) != AN5D_OK)
            return s;
        memset(out, 0, sizeof *out);
        out->ndim = p->ndim; out->rad = p->rad; out->bT = c.bT; out->vec = c.vec;
        for (int i = 0; i < p->ndim; ++i) out->interior[i] = dm.E[i] - 2 * p->rad;
        int64_t ntb = 1;
        for (int i = 0; i < p->ndim - 1; ++i) {
            out->bS[i] = g.C[i] + 2 * c.bT * p->rad;
            out->bS_loaded[i] = g.loaded[i];
            out->compute[i] = g.C[i];
            out->halo_loaded[i] = g.halo[i];
            out->n_tiles[i] = g.ntiles[i];
            ntb *= g.ntiles[i];
        }
        out->n_tb = ntb;
        out->h = g.h;
        out->n_stream_blocks = g.n_sb;
        out->n_tb_prime = g.n_sb * ntb;
        int64_t ov = 0;
        for (int T = 0; T < c.bT; ++T) ov += (int64_t)p->rad * (c.bT - T);
        out->stream_overlap = 2 * ov;
        out->n_thr = inst->threads;
        out->units_per_block = 1;
        out->grid_blocks = p->ndim == 2 ? std::min<int64_t>(g.n_units,
                                                            (int64_t)resident_blocks(*inst) * dev_info().n_sm)
                                        : g.n_units;
        out->n_units = run_frac() > 0
                           ? (int64_t)build_runs(p->ndim, g,
                                                 run_warps(p->ndim == 2 ? out->grid_blocks : resident_units(*inst)),
                                                 run_frac()).size()
                           : g.n_units;
        if (p->ndim == 3) out->grid_blocks = out->n_units * std::max(1, inst->cluster);
        out->smem_bytes = inst->smem_bytes;
        cudaFuncAttributes attr{};
        if (cudaFuncGetAttributes(&attr, inst->fn_interior) == cudaSuccess) out->regs_per_thread = attr.numRegs;
        else cudaGetLastError();
        return AN5D_OK;
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

an5d_status an5d_copy_ring(an5d_plan* p, const void* src, void* dst, const int64_t* extents, const int64_t* pitches,
                           int64_t outer_offset, int64_t global_outer_extent, void* stream) {
    try {
        if (!p || !src || !dst) return fail(AN5D_ERR_INVALID_ARGUMENT, "NULL argument");
        Dims dm{};
        an5d_status s = read_dims(*p, extents, pitches, dm);
        if (s != AN5D_OK) return s;
        return launch_copy(*p, src, dst, dm, true, outer_offset, global_outer_extent, (cudaStream_t)stream);
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

an5d_status an5d_sweep_peer(an5d_plan* p, const void* src, void* dst, const int64_t* extents, const int64_t* pitches,
                            int degree, const an5d_config* cfg, int64_t outer_offset, int64_t global_outer_extent,
                            int64_t out_lo, int64_t out_hi, const an5d_peer_store* peers, int32_t* debug_write_count,
                            void* stream) {
    try {
        if (!p || !cfg) return fail(AN5D_ERR_INVALID_ARGUMENT, "NULL argument");
        if (p->nf > 1 && peers) return fail(AN5D_ERR_UNSUPPORTED, "peer stores: single-field plans only");
        Dims dm{};
        an5d_status s = read_dims(*p, extents, pitches, dm);
        if (s != AN5D_OK) return s;
        if ((s = check_alignment(*p, src, dm, "src")) != AN5D_OK) return s;
        if ((s = check_alignment(*p, dst, dm, "dst")) != AN5D_OK) return s;
        if (degree < 1 || degree > cfg->bT) return fail(AN5D_ERR_INVALID_ARGUMENT, "degree must be in [1, bT]");
        if (global_outer_extent < dm.E[0] + outer_offset || outer_offset < 0)
            return fail(AN5D_ERR_INVALID_ARGUMENT, "slab outside the global array");
        // clip output planes to the global interior
        out_lo = std::max(out_lo, (int64_t)p->rad - outer_offset);
        out_hi = std::min(out_hi, global_outer_extent - p->rad - outer_offset);
        if (out_lo < 0 || out_hi > dm.E[0]) return fail(AN5D_ERR_INVALID_ARGUMENT, "output planes outside array");
        if (out_hi <= out_lo) return AN5D_OK;
        // the inputs the sweep needs must exist locally unless that side is the global face
        if (out_lo - (int64_t)degree * p->rad < 0 && outer_offset > 0)
            return fail(AN5D_ERR_INVALID_ARGUMENT, "slab lacks %d ghost planes below", degree * p->rad);
        if (out_hi + (int64_t)degree * p->rad > dm.E[0] && outer_offset + dm.E[0] < global_outer_extent)
            return fail(AN5D_ERR_INVALID_ARGUMENT, "slab lacks %d ghost planes above", degree * p->rad);
        if (peers) {
            for (int k = 0; k < 2; ++k) {
                if (peers->send_planes[k] < 0 || peers->send_planes[k] > out_hi - out_lo)
                    return fail(AN5D_ERR_INVALID_ARGUMENT, "send_planes[%d] outside the output planes", k);
                if (peers->peer_dst[k] && check_alignment(*p, peers->peer_dst[k], dm, "peer_dst") != AN5D_OK)
                    return AN5D_ERR_UNSUPPORTED;
            }
        }
        an5d_config c{};
        if ((s = resolve_config(*p, dm, 0, cfg, c)) != AN5D_OK) return s;
        if ((s = ensure_streams(*p)) != AN5D_OK) return s;
        return launch_sweep(*p, src, dst, dm, degree, c, outer_offset, global_outer_extent, out_lo, out_hi,
                            debug_write_count, peers, false, (cudaStream_t)stream);
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

an5d_status an5d_sweep(an5d_plan* p, const void* src, void* dst, const int64_t* extents, const int64_t* pitches,
                       int degree, const an5d_config* cfg, int64_t outer_offset, int64_t global_outer_extent,
                       int64_t out_lo, int64_t out_hi, int32_t* debug_write_count, void* stream) {
    return an5d_sweep_peer(p, src, dst, extents, pitches, degree, cfg, outer_offset, global_outer_extent, out_lo,
                           out_hi, nullptr, debug_write_count, stream);
}

// ---- stream-ordered flags and CUDA IPC (fused multi-GPU halo exchange plumbing) -----------------

an5d_status an5d_stream_signal(uint32_t* flag, uint32_t value, void* stream) {
    static StreamValue32Fn fn = driver_fn<StreamValue32Fn>("cuStreamWriteValue32");
    if (!flag) return fail(AN5D_ERR_INVALID_ARGUMENT, "flag is NULL");
    if (!fn) return fail(AN5D_ERR_CUDA, "cuStreamWriteValue32 not available");
    const CUresult r = fn((CUstream)stream, (CUdeviceptr)flag, value, 0 /* with a memory barrier */);
    return r == CUDA_SUCCESS ? AN5D_OK : fail(AN5D_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
}

an5d_status an5d_stream_wait(const uint32_t* flag, uint32_t value, void* stream) {
    static StreamValue32Fn fn = driver_fn<StreamValue32Fn>("cuStreamWaitValue32");
    if (!flag) return fail(AN5D_ERR_INVALID_ARGUMENT, "flag is NULL");
    if (!fn) return fail(AN5D_ERR_CUDA, "cuStreamWaitValue32 not available");
    const CUresult r = fn((CUstream)stream, (CUdeviceptr)flag, value, CU_STREAM_WAIT_VALUE_GEQ);
    return r == CUDA_SUCCESS ? AN5D_OK : fail(AN5D_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
}

an5d_status an5d_ipc_export(const void* ptr, void* handle, int64_t* offset) {
    static AddressRangeFn range = driver_fn<AddressRangeFn>("cuMemGetAddressRange");
    if (!ptr || !handle || !offset) return fail(AN5D_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!range) return fail(AN5D_ERR_CUDA, "cuMemGetAddressRange not available");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return fail(AN5D_ERR_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    memcpy(handle, &h, sizeof h);
    *offset = (int64_t)((CUdeviceptr)ptr - base);
    return AN5D_OK;
}

an5d_status an5d_ipc_open(const void* handle, void** base) {
    if (!handle || !base) return fail(AN5D_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    const cudaError_t e = cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? AN5D_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

an5d_status an5d_ipc_close(void* base) {
    const cudaError_t e = cudaIpcCloseMemHandle(base);
    return e == cudaSuccess ? AN5D_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

an5d_status an5d_run(an5d_plan* p, void* grid_in, void* grid_out, const int64_t* extents, const int64_t* pitches,
                     int64_t T, const an5d_config* cfg, void* stream) {
    try {
        if (!p) return fail(AN5D_ERR_INVALID_ARGUMENT, "plan is NULL");
        if (T < 0) return fail(AN5D_ERR_INVALID_ARGUMENT, "T < 0");
        Dims dm{};
        an5d_status s = read_dims(*p, extents, pitches, dm);
        if (s != AN5D_OK) return s;
        if ((s = check_alignment(*p, grid_in, dm, "grid_in")) != AN5D_OK) return s;
        if ((s = check_alignment(*p, grid_out, dm, "grid_out")) != AN5D_OK) return s;
        if (grid_in == grid_out) return fail(AN5D_ERR_INVALID_ARGUMENT, "grid_in and grid_out must differ");
        cudaStream_t st = (cudaStream_t)stream;
        p->launches = 0;
        if (T == 0) return launch_copy(*p, grid_in, grid_out, dm, false, 0, dm.E[0], st);
        an5d_config c{};
        if ((s = resolve_config(*p, dm, T, cfg, c)) != AN5D_OK) return s;
        if (p->comm) {   // NCCL slab mode (an5d_set_comm)
            if ((s = ensure_streams(*p)) != AN5D_OK) return s;
            return run_comm(*p, grid_in, grid_out, dm, T, c, st);
        }
        std::vector<int> deg;
        bool tc = false;
        make_schedule(T, c.bT, deg, tc);
        // validate every sweep's geometry before the first launch (no partial writes on error)
        for (int d : deg) {
            const Instance* inst = find_instance(*p, d, c);
            SweepGeom g{};
            if ((s = sweep_geometry(*p, *inst, dm, d, c.h, 0, dm.E[0], p->rad, dm.E[0] - p->rad, g)) != AN5D_OK)
                return s;
        }
        if ((s = ensure_streams(*p)) != AN5D_OK) return s;
        // both buffers carry the input ring (D1: the ring is never written by a sweep)
        if ((s = launch_copy(*p, grid_in, grid_out, dm, true, 0, dm.E[0], st)) != AN5D_OK) return s;
        void* bufs[2] = {grid_in, grid_out};
        for (size_t i = 0; i < deg.size(); ++i) {
            const void* src = bufs[i % 2];
            void* dst = bufs[(i + 1) % 2];
            if ((s = launch_sweep(*p, src, dst, dm, deg[i], c, 0, dm.E[0], p->rad, dm.E[0] - p->rad, nullptr, nullptr,
                                  false, st)) !=
                AN5D_OK)
                return s;
        }
        if (tc) {
            if ((s = launch_copy(*p, grid_in, grid_out, dm, false, 0, dm.E[0], st)) != AN5D_OK) return s;
        }
        return AN5D_OK;
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

an5d_status an5d_run_slab(an5d_plan* p, void* grid_in, void* grid_out, const int64_t* extents, const int64_t* pitches,
                          int64_t T, const an5d_config* cfg, int64_t outer_offset, int64_t global_outer_extent,
                          int64_t own_lo, int64_t own_hi, an5d_slab_links* links, void* stream) {
    try {
        if (!p || !links || !links->flag) return fail(AN5D_ERR_INVALID_ARGUMENT, "NULL argument");
        if (p->nf > 1) return fail(AN5D_ERR_UNSUPPORTED, "slab runs: single-field plans only");
        if (T < 0) return fail(AN5D_ERR_INVALID_ARGUMENT, "T < 0");
        Dims dm{};
        an5d_status s = read_dims(*p, extents, pitches, dm);
        if (s != AN5D_OK) return s;
        if ((s = check_alignment(*p, grid_in, dm, "grid_in")) != AN5D_OK) return s;
        if ((s = check_alignment(*p, grid_out, dm, "grid_out")) != AN5D_OK) return s;
        if (grid_in == grid_out) return fail(AN5D_ERR_INVALID_ARGUMENT, "grid_in and grid_out must differ");
        if (own_lo < 0 || own_hi > dm.E[0] || own_hi <= own_lo) return fail(AN5D_ERR_INVALID_ARGUMENT, "bad owned planes");
        for (int k = 0; k < 2; ++k)
            if (!links->peer_flag[k] != !links->peer_bufs[k][0] || !links->peer_bufs[k][0] != !links->peer_bufs[k][1])
                return fail(AN5D_ERR_INVALID_ARGUMENT, "side %d: buffers and flag must be given together", k);
        cudaStream_t st = (cudaStream_t)stream;
        an5d_config c{};
        if ((s = resolve_config(*p, dm, T, cfg, c)) != AN5D_OK) return s;
        std::vector<int> deg;
        bool tc = false;
        make_schedule(T, c.bT, deg, tc);
        for (int k = 0; k < 2; ++k)   // a neighbour needs b_T rad ghost planes from each side
            if (links->peer_flag[k] && (own_hi - own_lo) < (int64_t)c.bT * p->rad)
                return fail(AN5D_ERR_INVALID_ARGUMENT, "slab owns fewer planes than the ghost depth");
        if ((s = ensure_streams(*p)) != AN5D_OK) return s;
        // upload every sweep's run table now: a synchronous upload behind a stream wait on a
        // neighbour that has not been enqueued yet (one process, several slabs) could deadlock
        {
            const int64_t lo = std::max(own_lo, (int64_t)p->rad - outer_offset);
            const int64_t hi = std::min(own_hi, global_outer_extent - p->rad - outer_offset);
            for (size_t i = 0; i < deg.size() && hi > lo; ++i)
                if ((s = launch_sweep(*p, grid_in, grid_out, dm, deg[i], c, outer_offset, global_outer_extent, lo, hi,
                                      nullptr, nullptr, true, st)) != AN5D_OK)
                    return s;
        }
        p->launches = 0;
        if ((s = launch_copy(*p, grid_in, grid_out, dm, true, outer_offset, global_outer_extent, st)) != AN5D_OK) return s;
        void* bufs[2] = {grid_in, grid_out};
        for (size_t i = 0; i < deg.size(); ++i) {
            const void* src = bufs[i % 2];
            void* dst = bufs[(i + 1) % 2];
            const int par = (int)((i + 1) % 2);           // dst is grid_out (1) or grid_in (0)
            const int nd = i + 1 < deg.size() ? deg[i + 1] : 0;
            for (int k = 0; k < 2; ++k)
                if (links->peer_flag[k] &&
                    (s = an5d_stream_wait(links->peer_flag[k], links->epoch + (uint32_t)i, stream)) != AN5D_OK)
                    return s;
            an5d_peer_store ps{};
            for (int k = 0; k < 2; ++k)
                if (links->peer_flag[k] && nd) {
                    ps.peer_dst[k] = links->peer_bufs[k][par];
                    ps.peer_plane_shift[k] = links->peer_plane_shift[k];
                    ps.send_planes[k] = (int64_t)nd * p->rad;
                }
            if ((s = an5d_sweep_peer(p, src, dst, extents, pitches, deg[i], &c, outer_offset, global_outer_extent,
                                     own_lo, own_hi, &ps, nullptr, stream)) != AN5D_OK)
                return s;
            if ((s = an5d_stream_signal(links->flag, links->epoch + (uint32_t)i + 1, stream)) != AN5D_OK) return s;
        }
        links->epoch += (uint32_t)deg.size();
        if (tc) {   // b_T == 1 with an even sweep count: the owned planes' result is in grid_in
            const size_t off = (size_t)own_lo * dm.pitch[0] * p->elem, n = (size_t)(own_hi - own_lo) * dm.pitch[0] * p->elem;
            const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(grid_out) + off, static_cast<char*>(grid_in) + off, n,
                                                  cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "trailing copy");
        }
        return AN5D_OK;
    } catch (...) {
        return fail(AN5D_ERR_INVALID_ARGUMENT, "unexpected exception");
    }
}

}  // extern "C"
