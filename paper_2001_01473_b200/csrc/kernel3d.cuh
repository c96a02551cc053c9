// kernel3d.cuh -- N.5D (2.5D spatial + b_T temporal) blocked 3D stencil sweep for sm_100a.
//
// PAPER.md mapping (AN5D, arXiv 2001.01473):
//   * a thread block owns a (y, x) tile and streams along z, the outermost dimension (2.5D
//     blocking);
//   * b_T computational streams; level T works on plane s - T*rad (fig:tier);
//   * overlapped tiles with b_T*rad halos recomputed redundantly, compute region stored
//     (P:166-172);
//   * stream-dimension neighbours never touch shared memory: every arriving plane of level T-1
//     updates the 2*rad+1 in-flight output planes of level T held in registers (associative partial
//     sums; for star the off-centre planes add one tap);
//   * fixed register slots indexed by plane mod (2*rad+1), stream loop unrolled by that period
//     (P:384-389);
//   * in-plane neighbours of other threads go through a DOUBLE-BUFFERED shared-memory exchange with
//     one block barrier per level -- but only the rad rows a neighbour needs, not the
//     whole sub-plane;
//   * the boundary ring is never computed: ring planes / rows / cells that are the input of a level
//     take their original values, read back from the on-chip plane stage.
//
// B200 design:
//   * 256 threads = 16 (x) x 16 (y); thread (tx, ty) owns a VY x 4 patch (a 16-byte vector per row
//     for fp32, two for fp64); a tile plane is 64 x 16 VY cells;
//   * x neighbours: own registers + shuffles inside each 16-lane half-warp (2 rad per row); y
//     neighbours: own registers + rad rows from the threads above / below through shared memory;
//   * fp32 arithmetic in packed pairs (FFMA2/FMUL2) for every tap with an even x offset, scalar
//     FFMA for odd x offsets (see lane.cuh);
//   * level-0 planes staged by TMA (cp.async.bulk.tensor.3d, one elected thread, completion on one
//     mbarrier per stage slot) into a ring of D planes (prefetch distance PF, plus the (b_T-1)*rad
//     planes ring pinning reads back).  The hardware zero-fills the parts of the tile window that
//     leave the array (y, z, x past the end), so edge tiles stage exactly like interior ones;
//   * one block per (tile, stream block) unit; units whose tile window touches the x/y ring or the
//     array end are numbered first and run a separately instantiated EDGE copy of the stream loop
//     (the z ring / z array ends cost a uniform per-step check in both copies).
#pragma once
#include "args.hpp"
#include "common.cuh"
#include "lane.cuh"

namespace an5d {


constexpr int kPrefetch3D = 3;

// Thread layout (TXT_ x 16 threads, patch VY x VX_ cells per thread):
//   TXT_ = 16, VX_ = 4: 256 threads, 64 x 16 VY tile plane (the default; fp32 and fp64);
//   TXT_ = 32, VX_ = 2: 512 threads, 64 x 16 VY tile -- fp64 with half the registers per thread,
//                       so twice the warps per SM (one 16-byte vector per patch row);
//   TXT_ = 32, VX_ = 4: 512 threads, 128 x 16 VY tile -- a wider tile: less x-halo redundancy
//                       (the planner's b_S choice).
//   OS_ ("output-stationary" staging, bit flags):
//     bit 0 (y): the TMA box adds rad rows above and below the thread window, so level 1 reads
//                real rows there and the y halo the threads compute shrinks from b_T rad to
//                (b_T - 1) rad (any b_T; levels >= 2 exchange rows as before);
//     bit 1 (x): the box also adds the x halo (HXO cells left/right) and every thread reads its
//                level-1 x neighbours from the staged plane -- at b_T = 1 the threads then cover
//                only the compute region (kTX x kTY cells): no halo cell is computed, no shuffle
//                is needed; at b_T >= 2 levels >= 2 shuffle as before and the threads' x halo
//                shrinks to (b_T - 1) rad (rounded to vectors: pays for fp64, 2-cell vectors).
template <typename T, int R, int BT, int VY, int TXT_ = 16, int VX_ = 4, int OS_ = 0>
struct Kernel3DTraits {
    static constexpr int VX = VX_;
    static constexpr int TXT = TXT_, TYT = 16;
    static constexpr int OS = OS_;
    static constexpr bool OSY = (OS & 1) != 0, OSX = (OS & 2) != 0;
    static_assert(OSX || VX >= R, "x halo: a thread's rad neighbour cells must come from one adjacent thread");
    static_assert(!OSX || OSY, "x staging implies y staging");
    static_assert(VX % VecOf<T>::A == 0, "patch rows are whole 16-byte vectors");
    static_assert(!OSX || BT == 1 || VX >= R, "x staging at b_T >= 2: levels >= 2 still shuffle");
    static constexpr int kThreads = TXT * TYT;
    static constexpr int kTX = TXT * VX, kTY = TYT * VY;    // thread window, x by y
    static constexpr int HXO = OSX ? ((R + VecOf<T>::A - 1) / VecOf<T>::A) * VecOf<T>::A : 0;  // staged x halo
    // XPAIR (fp32, no x staging, b_T rad = 2 mod 4): the loaded x halo is b_T rad itself instead of
    // b_T rad rounded up to a 16-byte vector, so the compute width is kTX - 2 b_T rad (b_T 2, rad 1:
    // 60 instead of 56 -- at 512^3 9 x tiles instead of 10).  A TMA box must start on a 16-byte x
    // boundary (an unaligned start faults: profiles/r02z_xpair_probe_unaligned_tma.txt), so the box
    // starts XOFF = 2 cells before the window and is 4 cells wider; threads read their patch XOFF
    // cells into the staged row (8-byte shared loads) and store 8-byte cell pairs (every patch and
    // every compute region then starts 2 cells off a 16-byte boundary; the compute width is a
    // multiple of 4).  Other halos keep the rounding.
    static constexpr bool XPAIR = sizeof(T) == 4 && HXO == 0 && (BT * R) % 4 == 2;
    static constexpr int XOFF = XPAIR ? 2 : 0;              // staged column of the window's first cell
    static constexpr int SG = XPAIR ? 2 : VecOf<T>::A;       // store granule (cells)
    static constexpr int kTXW = kTX + 2 * HXO;              // loaded window (cells)
    static constexpr int kTXL = kTXW + 2 * XOFF;            // staged row = TMA box width (= kTX unless OS / XPAIR)
    static constexpr int kTYL = kTY + (OSY ? 2 * R : 0);    // loaded rows
    static constexpr int PROWS = kTY + 2 * R;               // staged rows (R pad rows per side; OS: halo rows)
    // elements per staged plane, rounded to 128 bytes: every slot is a TMA destination, which must
    // be 128-byte aligned (the output-stationary 72-wide rows broke that: misaligned address)
    static constexpr int PLANE = ((PROWS * kTXL * (int)sizeof(T) + 127) / 128) * 128 / (int)sizeof(T);
    static constexpr int XROW = kTXL;                       // exchange row (cells)
    // y-halo exchange: a thread publishes the rad rows its neighbours need (top and bottom rad rows
    // of its patch) -- possible while rad <= VY; otherwise (rad > VY) it publishes its whole patch
    // into a padded plane and reads rad rows spanning several threads above / below
    static constexpr bool XPLANE = R > VY;
    static constexpr int XBAND = 2 * R * XROW;              // exchange rows of one thread row
    static constexpr int XBUF = XPLANE ? PROWS * kTXL : (TYT + 2) * XBAND;  // one exchange buffer
    // Level skew SK (see sweep3d_unit): with SK = 1 level L at step s takes the plane level L-1
    // completed at step s-1, so all levels' halo rows are exchanged together behind the one
    // barrier a step has anyway (1 barrier per plane instead of b_T).  Costs deeper staging (the
    // arrival of level L is (L-1)(rad+1) planes old) and an exchange buffer per level.  Off for
    // rotated-slot kernels and where the shared memory would not fit.
    static constexpr int D0 = kPrefetch3D + (BT - 1) * R + 1;                       // SK = 0
    static constexpr int D1 = kPrefetch3D + (BT >= 2 ? (BT - 2) * (R + 1) + R : 0) + 1;  // SK = 1
    // D staged planes, nxb exchange buffers, D mbarriers (one per stage slot)
    static constexpr size_t smem_of(int d, int nxb) {
        return ((size_t)d * PLANE + (size_t)nxb * XBUF) * sizeof(T) + (size_t)d * 8;
    }
    static constexpr size_t kSmem1 = smem_of(D1, 2 * (BT - 1));
#ifndef AN5D_SK3D
    static constexpr int SK = (BT >= 2 && kSmem1 <= 220 * 1024) ? 1 : 0;
#else
    static constexpr int SK = AN5D_SK3D && BT >= 2 && kSmem1 <= 220 * 1024;
#endif
    static constexpr int D = SK ? D1 : D0;                  // staged planes
    static constexpr int NXB = SK ? 2 * (BT - 1) : 2;       // exchange buffers
    static constexpr size_t kSmemBytes = smem_of(D, NXB);
    // XPAIR rows are kTXL = kTX + 4 cells, so a layout whose TMA box lands R rows into the slot
    // (no cluster, no y staging) would put the box off the 128-byte boundary TMA destinations need
    // (misaligned address): the whole shared-memory layout then starts LEAD cells late, with
    // LEAD + R kTXL = 0 mod 32 cells (slots stay multiples of 128 bytes)
    static constexpr int lead(int cl) {
        return (XPAIR && !(cl > 1 || OSY)) ? (32 - (R * kTXL) % 32) % 32 : 0;
    }
    static constexpr size_t smem_total(int cl) { return kSmemBytes + (size_t)lead(cl) * sizeof(T); }
};

// unit -> (tile y, tile x, stream block): frame tiles (those that can touch the ring or the array
// end: first and last two in each direction) of every stream block first, then the interior
// tiles in stream-block order 0, n_sb-1, 1, 2, ...
__device__ __forceinline__ void unit_to_tile3d(const Sweep3DArgs& a, int64_t u, int& ty, int& tx, int64_t& sb) {
    const int ny = a.nty, nx = a.ntx;
    if (ny < 4 || nx < 4) {
        const int64_t NT = (int64_t)ny * nx;
        sb = u / NT;
        const int t = (int)(u % NT);
        ty = t / nx;
        tx = t % nx;
        return;
    }
    const int F = 3 * nx + (ny - 3) * 3;   // frame tiles
    if (u < (int64_t)F * a.n_sb) {
        sb = u / F;
        int f = (int)(u % F);
        if (f < 3 * nx) {
            const int r = f / nx;
            ty = r == 0 ? 0 : ny - r;
            tx = f % nx;
        } else {
            f -= 3 * nx;
            ty = 1 + f / 3;
            const int c = f % 3;
            tx = c == 0 ? 0 : nx - c;
        }
        return;
    }
    const int64_t v = u - (int64_t)F * a.n_sb;
    const int64_t ni = (int64_t)(ny - 3) * (nx - 3);
    const int64_t sbi = v / ni;
    const int t = (int)(v % ni);
    sb = sbi == 0 ? 0 : (sbi == 1 ? a.n_sb - 1 : sbi - 1);
    ty = 1 + t / (nx - 3);
    tx = 1 + t % (nx - 3);
}

struct Unit3D {
    int cy0, cy1, cx0, cx1;      // compute region
    int wy0, wx0;                // loaded window origin
    int64_t p0, p1;              // output planes
    int64_t s_first, s_end, s_a, s_b;
    bool ring_xy;                // window touches the y/x ring or array end
};

template <typename T, int R>
using Coeffs3D = Coeffs<typename CoefElem<T>::type, (2 * R + 1) * (2 * R + 1) * (2 * R + 1) + (2 * R + 1) * (2 * R + 1)>;
// Entries [0, W^3): the dense table (fp32: broadcast pairs); W^3 + (dz+R) W + (dy+R), fp32 only:
// the mixed pair (c[dz][dy][+1], c[dz][dy][-1]) for the swapped-operand FFMA2 of the dx = +-1
// taps (see kernel2d.cuh Coeffs2D).

// CL > 1 (NEXT N2, thread-block-cluster halo sharing): the CL thread blocks of a cluster stack
// their tile windows along y and form ONE tall tile of CL x kTY rows: the y halo of b_T rad rows is
// loaded and recomputed only at the cluster's outer rows.  At a block's inner boundary the rows
// the neighbour owns come from the neighbour's shared memory (DSMEM): level 1 from its staged
// plane, level L >= 2 from its exchange buffer; the per-step block barrier becomes a cluster
// barrier (release/acquire), which also orders the neighbour's reads against the reuse of its
// stage slots and exchange buffers (both are double-buffered or D - PF >= 1 planes deep).
template <typename T, int R, int BT, int VY, bool BOX, bool EDGE, int TXT, int VX_, int CL = 1, int OS = 0>
__device__ __forceinline__ void sweep3d_unit(const Sweep3DArgs& a, const Coeffs3D<T, R>& cf, T* const smem,
                                             const Unit3D& g, const void* tmap, const unsigned crank = 0) {
    using K = Kernel3DTraits<T, R, BT, VY, TXT, VX_, OS>;
    static_assert(!OS || CL == 1, "output-stationary tiles are not clustered");
    static_assert(CL == 1 || !K::XPLANE, "cluster halo sharing needs rad <= VY (row-band exchange)");
    // Cluster synchronisation.  Every block stages R extra rows above and below its window (the
    // TMA box is kTY + 2R rows), so level 1 never reads a neighbour; levels >= 2 read the
    // neighbours' exchange buffers.  With the level skew (SK, one exchange per step) the cluster
    // barrier is SPLIT: arrive right after a step's publish (before its global stores), wait at
    // the next step's start -- the stores and the TMA wait overlap the barrier latency (a joined
    // release barrier per step waited for the step's stores and measured 2x slower, r02e).
    // Without the skew (b_T >= 2) each level's exchange takes a full cluster barrier; b_T = 1 has
    // no exchange at all (block barriers only).
    constexpr bool CSPLIT = CL > 1 && K::SK && !(BOX && R >= 2);
    constexpr bool CFULL = CL > 1 && !CSPLIT && BT >= 2;
    auto block_sync = [&]() {
        if constexpr (CFULL) cluster_sync_all();
        else __syncthreads();
    };
    [[maybe_unused]] const bool peer_up = CL > 1 && crank > 0;          // block above in the cluster
    [[maybe_unused]] const bool peer_dn = CL > 1 && crank + 1 < (unsigned)CL;   // block below
    using LN = Lane<T, K::VX>;
    using E = typename LN::E;
    constexpr int NE = LN::NE;              // elements per patch row
    constexpr int VX = K::VX, A = VecOf<T>::A, NCH = VX / A;
    constexpr int P = 2 * R + 1, W = 2 * R + 1;
    constexpr int D = K::D, PF = kPrefetch3D;
    // High-order box stencils ((2 rad+1)^3 >= 125 taps per cell): unrolling the stream loop by the
    // slot period P would multiply an already huge loop body by P (compile time, I-cache), so the
    // slots are rotated instead: 2*rad moves per cell and step against >= 125 FMAs.
    constexpr bool ROT = BOX && R >= 2;
    // fp32 box rad 4 (729 taps): the per-plane contributions run as a runtime loop (see the level
    // body).  Measured on B200 (profiles/r02d_boxhi.jsonl): box3d4r fp32 12.2 -> 18.3 GCells/s;
    // box3d3r fp32 -9 %, fp64 box3d3r -14 % and box3d4r -55 % (the rotation spills at 255
    // registers), so those keep the static unroll.
#ifdef AN5D_RLOOP_MIN_R
    constexpr bool RLOOP = ROT && R >= AN5D_RLOOP_MIN_R;
#else
    constexpr bool RLOOP = ROT && R >= 4 && sizeof(T) == 4;
#endif
    constexpr int U = ROT ? 1 : P;          // unroll factor of the stream loop
    // level skew (traits): SK = 1 -> level L at step s consumes level L-1's plane of step s-1;
    // levels run top-down inside a step (a level reads its arrival slot before the level below
    // recycles it); every level's halo rows travel through one exchange per step
    constexpr int SK = (K::SK && !ROT) ? 1 : 0;
    // (a rotated-slot kernel runs unskewed inside the skewed traits' buffers: D1 >= D0, >= 2 buffers)
    constexpr int DL = R + SK;              // plane delay per level
    constexpr int kTX = K::kTXL;   // staged row stride (the loaded width)

    T* __restrict__ dst = static_cast<T*>(a.dst);
    const int tid = threadIdx.x;
    const int txi = tid % K::TXT, tyi = tid / K::TXT;
    const int xs = K::HXO + txi * VX, ys = tyi * VY;    // patch origin in the tile window (OS: past the x halo)
    const int gy0 = g.wy0 + ys + (K::OSY ? R : 0), gx0 = g.wx0 + xs;   // this thread's first cell (array coords)
    T* const stage = smem;                              // D planes of PROWS x kTX
    T* const xch = smem + (size_t)D * K::PLANE;         // 2 exchange buffers
    const int own = (ys + R) * kTX + xs;                // patch origin inside a staged plane
    const int own_st = own + K::XOFF;                   // ... of the staged (TMA) plane itself (XPAIR)

    // per-thread masks (EDGE): ring cells, store coverage (st_full: whole store granules of SG
    // cells -- 16-byte vectors, or 8-byte pairs for XPAIR tiles)
    constexpr int SG = K::SG, NSG = VX / SG;
    unsigned ring_mask = 0, st_full = 0, st_elem = 0;
#pragma unroll
    for (int yy = 0; yy < VY; ++yy) {
        const int y = gy0 + yy;
        const bool yin = y >= 0 && y < a.Ey;
#pragma unroll
        for (int j = 0; j < NSG; ++j) {
            const int x = gx0 + j * SG;
            if (y >= g.cy0 && y < g.cy1 && x >= g.cx0 && x + SG <= g.cx1) st_full |= 1u << (yy * NSG + j);
        }
        if constexpr (EDGE) {
#pragma unroll
            for (int xx = 0; xx < VX; ++xx) {
                const int x = gx0 + xx;
                const bool in = yin && x >= 0 && x < a.Ex;
                const bool ring = y < R || y >= a.Ey - R || x < R || x >= a.Ex - R;
                if (in && ring) ring_mask |= 1u << (yy * VX + xx);
                if (!((st_full >> (yy * NSG + xx / SG)) & 1u) && y >= g.cy0 && y < g.cy1 && x >= g.cx0 && x < g.cx1)
                    st_elem |= 1u << (yy * VX + xx);
            }
        }
    }

    // ---- level-0 staging: one TMA box {kTX, kTY, 1} per plane, issued by thread 0 -------------------
    // Planes outside [s_a, s_b) are not loaded (they feed nothing that is stored or pinned): the
    // slot's barrier is completed by a plain arrive.
    uint64_t* const mbar = reinterpret_cast<uint64_t*>(smem + (size_t)D * K::PLANE + (size_t)K::NXB * K::XBUF);
    // box rows: kTY (+ the R pad rows above and below with clusters: level 1 stays local)
    constexpr int kBoxRows = K::kTY + ((CL > 1 || K::OSY) ? 2 * R : 0);
    constexpr unsigned kBoxBytes = (unsigned)(K::kTXL * kBoxRows * sizeof(T));
    auto issue_plane = [&](int64_t q, int slot) {
        if (tid == 0) {
            if (q >= g.s_a && q < g.s_b) {
                mbar_arrive_expect_tx(mbar + slot, kBoxBytes);
                tma_load_3d(stage + (size_t)slot * K::PLANE + ((CL > 1 || K::OSY) ? 0 : R * kTX), tmap,
                            g.wx0 - K::XOFF + a.x_off,
                            g.wy0 - (CL > 1 ? R : 0), (int)q, mbar + slot);
            } else {
                mbar_arrive(mbar + slot);
            }
        }
    };
    unsigned phase = 0;   // bit d: parity of the next completion of slot d's barrier
    auto wait_plane = [&](int slot) {
        mbar_wait(mbar + slot, (phase >> slot) & 1u);
        phase ^= 1u << slot;
    };
    // a patch row (VX cells) of a staged/exchange row pointer -> elements
    auto load_row = [&](E (&P_)[NE], const T* p) {
        T c[VX];
#pragma unroll
        for (int j = 0; j < NCH; ++j) ld_vec_shared<T>(c + j * A, p + j * A);
        LN::from_cells(P_, c);
    };
    // a patch row of a STAGED plane: XPAIR rows are 8-byte (not 16-byte) aligned
    auto load_row_st = [&](E (&P_)[NE], const T* p) {
        if constexpr (K::XPAIR) {
            T c[VX];
#pragma unroll
            for (int j = 0; j < VX; j += 2) {
                const float2 v = *reinterpret_cast<const float2*>(p + j);
                c[j] = v.x;
                c[j + 1] = v.y;
            }
            LN::from_cells(P_, c);
        } else {
            load_row(P_, p);
        }
    };
    auto store_row = [&](T* p, const E (&P_)[NE]) {
        T c[VX];
        LN::to_cells(c, P_);
#pragma unroll
        for (int j = 0; j < NCH; ++j) st_vec_shared<T>(p + j * A, c + j * A);
    };
    // a patch row of a neighbour block of the cluster: the same shared-memory offset in CTA `rank`
    [[maybe_unused]] auto load_row_peer = [&](E (&P_)[NE], const T* p, unsigned rank) {
        load_row(P_, map_cta(p, rank));
    };

    // ---- register state ---------------------------------------------------------------------------
    E acc[BT][P][VY][NE];
#pragma unroll
    for (int l = 0; l < BT; ++l)
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                for (int e = 0; e < NE; ++e) acc[l][k][yy][e] = E{};

    const int64_t s_a = g.s_a;
    const int64_t base0 = s_a - (s_a % P);
    auto rel = [&](int64_t x) -> int { return (int)max(min(x - base0, (int64_t)(1 << 30)), -(int64_t)(1 << 30)); };
    const int ra = rel(g.s_a), rb = rel(g.s_b);
    const int rlo = rel((int64_t)R - a.g_off), rhi = rel(a.gEz - R - a.g_off);
    const int rp0 = rel(g.p0), rp1 = rel(g.p1);

    if (tid == 0) {
        for (int d = 0; d < D; ++d) mbar_init(mbar + d, 1);
        mbar_fence_init();
    }
    __syncthreads();
#pragma unroll
    for (int d = 0; d < PF; ++d) issue_plane(base0 + d, d);
    if constexpr (CSPLIT) cluster_arrive();   // phase 0: matched by the first step's wait

    // pin plane qi (relative index) of a patch to its original ring values, read from the stage
    auto pin = [&](E (&u)[VY][NE], int qi) {
        if (qi < ra || qi >= rb) return;                  // not in the array: feeds nothing kept
        const T* sq = stage + (size_t)(qi % D) * K::PLANE + own_st;
        if (qi < rlo || qi >= rhi) {                      // z-ring plane: every cell
#pragma unroll
            for (int yy = 0; yy < VY; ++yy) load_row_st(u[yy], sq + yy * kTX);
        } else if (EDGE && g.ring_xy && ring_mask) {      // x/y-ring cells of this thread
#pragma unroll
            for (int yy = 0; yy < VY; ++yy) {
                E o[NE];
                load_row_st(o, sq + yy * kTX);
#pragma unroll
                for (int xx = 0; xx < VX; ++xx) {
                    T& uc = LN::cell(u[yy], xx);
                    uc = ((ring_mask >> (yy * VX + xx)) & 1u) ? LN::cell(o, xx) : uc;
                }
            }
        }
    };
    // publish the rows of patch u the threads above / below need; read theirs back
    auto publish = [&](T* xw, const E (&u)[VY][NE]) {
        if constexpr (!K::XPLANE) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                store_row(xw + (tyi + 1) * K::XBAND + r * kTX + xs, u[r]);                 // top rows
                store_row(xw + (tyi + 1) * K::XBAND + (R + r) * kTX + xs, u[VY - R + r]);  // bottom rows
            }
        } else {
#pragma unroll
            for (int yy = 0; yy < VY; ++yy) store_row(xw + own + yy * kTX, u[yy]);
        }
    };
    auto read_halo = [&](const T* xw, E (&lo)[R][NE], E (&hi)[R][NE]) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if constexpr (!K::XPLANE) {
                // cluster: the top thread row's "above" is the bottom thread row (band TYT) of the
                // block above, the bottom thread row's "below" the top thread row (band 1) below
                if (CL > 1 && tyi == 0 && peer_up)
                    load_row_peer(lo[r], xw + K::TYT * K::XBAND + (R + r) * kTX + xs, crank - 1);
                else
                    load_row(lo[r], xw + tyi * K::XBAND + (R + r) * kTX + xs);     // above: its bottom rows
                if (CL > 1 && tyi == K::TYT - 1 && peer_dn)
                    load_row_peer(hi[r], xw + 1 * K::XBAND + r * kTX + xs, crank + 1);
                else
                    load_row(hi[r], xw + (tyi + 2) * K::XBAND + r * kTX + xs);     // below: its top rows
            } else {
                load_row(lo[r], xw + own + (r - R) * kTX);
                load_row(hi[r], xw + own + (VY + r) * kTX);
            }
        }
    };

    int i = 0;          // step counter since base0
    int slot_i = 0;     // i mod D
    // element offset of this thread's patch in the plane the current step stores (advanced by one
    // plane per step: no 64-bit multiplies in the store path)
    int64_t st_off = (base0 - (int64_t)(BT - 1) * DL - R) * a.pz + (int64_t)gy0 * a.py + gx0;
    int xb = 0;         // exchange buffer parity
    const int64_t s_stop = g.s_end + (int64_t)(BT - 1) * SK;
    for (int64_t base = base0; base < s_stop; base += U) {
        static_for<0, U>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            const int64_t s = base + k;
            const int si = i;
            wait_plane(slot_i);                                // plane s has landed (TMA, mbarrier)
            if constexpr (CSPLIT) cluster_wait();              // ... every thread of the cluster published step s-1
            else block_sync();                                 // ... and every thread is past step s-1
            {
                int ns = slot_i + PF;
                if (ns >= D) ns -= D;
                issue_plane(s + PF, ns);   // planes outside [s_a, s_b): no traffic
            }
            const T* cur = stage + (size_t)slot_i * K::PLANE;
            ++i;
            if (++slot_i == D) slot_i = 0;
            // does any level's arrival need pinning this step?  z-ring planes (any unit, a few steps
            // at the ends of the array) or x/y-ring cells (EDGE units, every step).  SK = 1 pins at
            // completion (end of step) the planes p = si - (l-1) DL - R, l < b_T.
            const bool step_pin = (EDGE && g.ring_xy) ||
                                  (SK ? (si - (BT - 2) * DL - R < rlo || si - R >= rhi)
                                      : (si - (BT - 1) * R < rlo || si - R >= rhi));

            E u0[VY][NE];   // level-1 arrival (the staged plane s)
            static_for<1, BT + 1>([&](auto lc) {
                constexpr int L = SK ? BT + 1 - decltype(lc)::value : decltype(lc)::value;
                E (&u)[VY][NE] = [&]() -> E (&)[VY][NE] {
                    if constexpr (L == 1) return u0;
                    else return acc[L - 2][ROT ? 0 : pmod(k - SK - (L - 2) * DL - R, P)];
                }();
                // halo rows above / below the patch (y), as elements
                E yh_lo[R][NE], yh_hi[R][NE];
                if constexpr (L == 1) {
#pragma unroll
                    for (int yy = 0; yy < VY; ++yy) load_row_st(u0[yy], cur + own_st + yy * kTX);
#pragma unroll
                    for (int r = 0; r < R; ++r) {   // (clusters: the staged pad rows are real rows)
                        load_row_st(yh_lo[r], cur + own_st + (r - R) * kTX);
                        load_row_st(yh_hi[r], cur + own_st + (VY + r) * kTX);
                    }
                } else if constexpr (SK) {
                    // halo rows of level L-1's plane of the previous step, exchanged at its end
                    read_halo(xch + (size_t)(xb * (BT - 1) + (L - 2)) * K::XBUF, yh_lo, yh_hi);
                } else {
                    if (step_pin) pin(u, si - (L - 1) * R);
                    // publish the rad rows the threads above / below need, one barrier, read theirs
                    T* xw = xch + (size_t)xb * K::XBUF;
                    xb ^= 1;
                    publish(xw, u);
                    block_sync();
                    read_halo(xw, yh_lo, yh_hi);
                }
                // x halo of a row: rad cells from the left / right thread of the 16-lane segment
                auto xhalo = [&](const E (&row)[NE], T (&hl)[R], T (&hh)[R]) {
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        hh[m] = __shfl_down_sync(0xffffffffu, LN::cell(row, m), 1, K::TXT);
                        hl[m] = __shfl_up_sync(0xffffffffu, LN::cell(row, VX - R + m), 1, K::TXT);
                    }
                };
                // extended row accessor: row index yr in [-R, VY+R), cell c in [-R, VX+R)
                auto rowref = [&](int yr) -> const E (&)[NE] {
                    return yr < 0 ? yh_lo[yr + R] : (yr >= VY ? yh_hi[yr - VY] : u[yr]);
                };
                constexpr int XR = BOX ? VY + 2 * R : VY;       // rows needing an x halo
                T hl[XR][R], hh[XR][R];
                if constexpr (K::OSX && L == 1) {
                    // output-stationary (b_T = 1, level 1 = the staged plane): the rad cells left
                    // and right of each row, read from the stage as whole 16-byte vectors
                    constexpr int NVA = K::HXO;          // cells loaded per side (rad rounded to vectors)
#pragma unroll
                    for (int t = 0; t < XR; ++t) {
                        const T* rowp = cur + own + (BOX ? t - R : t) * kTX;
                        T lb[NVA], rb[NVA];
#pragma unroll
                        for (int j = 0; j < NVA; j += A) {
                            ld_vec_shared<T>(lb + j, rowp - NVA + j);
                            ld_vec_shared<T>(rb + j, rowp + VX + j);
                        }
#pragma unroll
                        for (int m = 0; m < R; ++m) {
                            hl[t][m] = lb[NVA - R + m];
                            hh[t][m] = rb[m];
                        }
                    }
                } else {
#pragma unroll
                for (int t = 0; t < XR; ++t) xhalo(rowref(BOX ? t - R : t), hl[t], hh[t]);
                }
                auto X = [&](int yr, int c) -> T {
                    const int t = BOX ? yr + R : yr;
                    return c < 0 ? hl[t][c + R] : (c >= VX ? hh[t][c - VX] : LN::cell(rowref(yr), c));
                };
                // contributions of arriving plane q = s - (L-1) R to output planes p = q - dz
                if constexpr (RLOOP) {
                    // high-order box: a RUNTIME loop over the 2 rad + 1 output planes (the static
                    // unroll is 5-12k instructions per plane: instruction-fetch bound, ncu
                    // r02b_ncu_b3d4r_f32: 53 % "no instruction" stalls).  The target plane is
                    // always slot 0; the slots rotate by one after each plane (P rotations = the
                    // identity), recycled slots start at zero (no first-tap multiply), and the
                    // taps of plane dz = R - j come from the parameter bank with a runtime offset.
#pragma unroll 1
                    for (int j = 0; j < P; ++j) {
                        const E* cz = &cf.c[(2 * R - j) * W * W];
                        auto tap_to = [&](E (&tgt)[VY][NE], const E c, int dy, int dx) {
#pragma unroll
                            for (int yy = 0; yy < VY; ++yy) {
                                if constexpr (sizeof(T) == 8) {
#pragma unroll
                                    for (int e = 0; e < NE; ++e) tgt[yy][e] = LN::fma(c, X(yy + dy, e + dx), tgt[yy][e]);
                                } else if ((dx & 1) == 0) {
#pragma unroll
                                    for (int e = 0; e < NE; ++e) {
                                        const int jj = 2 * e + dx;
                                        const E q = (jj >= 0 && jj + 1 < VX) ? rowref(yy + dy)[jj >> 1]
                                                                             : make_float2(X(yy + dy, jj), X(yy + dy, jj + 1));
                                        tgt[yy][e] = LN::fma(c, q, tgt[yy][e]);
                                    }
                                } else {
#pragma unroll
                                    for (int e = 0; e < NE; ++e) {
                                        tgt[yy][e].x = fmaf(c.x, X(yy + dy, 2 * e + dx), tgt[yy][e].x);
                                        tgt[yy][e].y = fmaf(c.x, X(yy + dy, 2 * e + 1 + dx), tgt[yy][e].y);
                                    }
                                }
                            }
                        };
                        const E* cmix = &cf.c[W * W * W + (2 * R - j) * W];
#pragma unroll
                        for (int dy = -R; dy <= R; ++dy)
#pragma unroll
                            for (int dx = -R; dx <= R; ++dx) {
                                if constexpr (sizeof(T) == 4) {
                                    if (dx == 1) continue;
                                    if (dx == -1) {   // dx = -1 and +1 together (swapped-operand FFMA2)
                                        const E cm = cz[(dy + R) * W + R - 1], cp = cz[(dy + R) * W + R + 1];
                                        const E mix = cmix[dy + R];
#pragma unroll
                                        for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                                            for (int e = 0; e < NE; ++e) {
                                                E& o = acc[L - 1][0][yy][e];
                                                const E q = rowref(yy + dy)[e];
                                                o.x = fmaf(cm.x, X(yy + dy, 2 * e - 1), o.x);
                                                o.y = fmaf(cp.x, X(yy + dy, 2 * e + 2), o.y);
                                                o = LN::fma(mix, make_float2(q.y, q.x), o);
                                            }
                                        continue;
                                    }
                                }
                                tap_to(acc[L - 1][0], cz[(dy + R) * W + (dx + R)], dy, dx);
                            }
                        // rotate the slots left by one: the next plane's target moves to slot 0
                        E t0[VY][NE];
#pragma unroll
                        for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                            for (int e = 0; e < NE; ++e) t0[yy][e] = acc[L - 1][0][yy][e];
#pragma unroll
                        for (int jj = 0; jj + 1 < P; ++jj)
#pragma unroll
                            for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                                for (int e = 0; e < NE; ++e) acc[L - 1][jj][yy][e] = acc[L - 1][jj + 1][yy][e];
#pragma unroll
                        for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                            for (int e = 0; e < NE; ++e) acc[L - 1][P - 1][yy][e] = t0[yy][e];
                    }
                } else
                static_for<0, 2 * R + 1>([&](auto dc) {
                    constexpr int dz = R - decltype(dc)::value;
                    constexpr int slot = ROT ? R - dz : pmod(k - (L - 1) * DL - dz, P);
                    auto tap = [&](const E c, int dy, int dx, bool first) {
#pragma unroll
                        for (int yy = 0; yy < VY; ++yy) {
                            if constexpr (sizeof(T) == 8) {
#pragma unroll
                                for (int e = 0; e < NE; ++e) {
                                    const T q = X(yy + dy, e + dx);
                                    acc[L - 1][slot][yy][e] = first ? LN::mul(c, q) : LN::fma(c, q, acc[L - 1][slot][yy][e]);
                                }
                            } else {
                                if ((dx & 1) == 0) {
#pragma unroll
                                    for (int e = 0; e < NE; ++e) {
                                        const int j = 2 * e + dx;
                                        const E q = (j >= 0 && j + 1 < VX) ? rowref(yy + dy)[j >> 1]
                                                                           : make_float2(X(yy + dy, j), X(yy + dy, j + 1));
                                        acc[L - 1][slot][yy][e] =
                                            first ? LN::mul(c, q) : LN::fma(c, q, acc[L - 1][slot][yy][e]);
                                    }
                                } else {
#pragma unroll
                                    for (int e = 0; e < NE; ++e) {
                                        E& o = acc[L - 1][slot][yy][e];
                                        o.x = first ? c.x * X(yy + dy, 2 * e + dx) : fmaf(c.x, X(yy + dy, 2 * e + dx), o.x);
                                        o.y = first ? c.x * X(yy + dy, 2 * e + 1 + dx)
                                                    : fmaf(c.x, X(yy + dy, 2 * e + 1 + dx), o.y);
                                    }
                                }
                            }
                        }
                    };
                    auto C = [&](int dy, int dx) { return cf.c[((dz + R) * W + (dy + R)) * W + (dx + R)]; };
                    // dx = -1 and +1 of one row together (fp32): outer products scalar, inner ones
                    // one FFMA2 on the pair with swapped halves (kernel2d.cuh Coeffs2D)
                    [[maybe_unused]] auto tap_pm1 = [&](int dy, bool first) {
                        if constexpr (sizeof(T) == 4) {
                            const E cm = C(dy, -1), cp = C(dy, 1), mix = cf.c[W * W * W + (dz + R) * W + (dy + R)];
#pragma unroll
                            for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                                for (int e = 0; e < NE; ++e) {
                                    E& o = acc[L - 1][slot][yy][e];
                                    const E q = rowref(yy + dy)[e];
                                    o.x = first ? cm.x * X(yy + dy, 2 * e - 1) : fmaf(cm.x, X(yy + dy, 2 * e - 1), o.x);
                                    o.y = first ? cp.x * X(yy + dy, 2 * e + 2) : fmaf(cp.x, X(yy + dy, 2 * e + 2), o.y);
                                    o = LN::fma(mix, make_float2(q.y, q.x), o);
                                }
                        }
                    };
                    constexpr bool PM1 = sizeof(T) == 4;
                    if constexpr (BOX) {
#pragma unroll
                        for (int dy = -R; dy <= R; ++dy)
#pragma unroll
                            for (int dx = -R; dx <= R; ++dx) {
                                if (PM1 && dx == 1) continue;
                                if (PM1 && dx == -1) tap_pm1(dy, dz == -R && dy == -R && R == 1);
                                else tap(C(dy, dx), dy, dx, dz == -R && dy == -R && dx == -R);
                            }
                    } else if constexpr (dz != 0) {
                        tap(C(0, 0), 0, 0, dz == -R);
                    } else {
                        // in-plane cross in lexicographic (dy, dx) order
#pragma unroll
                        for (int dy = -R; dy < 0; ++dy) tap(C(dy, 0), dy, 0, false);
#pragma unroll
                        for (int dx = -R; dx <= R; ++dx) {
                            if (PM1 && dx == 1) continue;
                            if (PM1 && dx == -1) tap_pm1(0, false);
                            else tap(C(0, dx), 0, dx, false);
                        }
#pragma unroll
                        for (int dy = 1; dy <= R; ++dy) tap(C(dy, 0), dy, 0, false);
                    }
                });
            });
            if constexpr (SK) {
                // completed planes of levels 1..b_T-1: pin (ring), then publish their halo rows for
                // the next step's levels 2..b_T; the next step's barrier orders the exchange
                const int wb = xb ^ 1;
                static_for<1, BT>([&](auto lc) {
                    constexpr int l = decltype(lc)::value;
                    auto& done = acc[l - 1][pmod(k - (l - 1) * DL - R, P)];
                    if (step_pin) pin(done, si - (l - 1) * DL - R);
                    publish(xch + (size_t)(wb * (BT - 1) + (l - 1)) * K::XBUF, done);
                });
                xb = wb;
                if constexpr (CSPLIT) cluster_arrive();   // published: the neighbours may read it next step
            }
            // ---- STORE level BT plane p = s - (BT-1) DL - R, compute region only --------------------
            const int pi = si - (BT - 1) * DL - R;
            if (pi >= rp0 && pi < rp1) {
                const int64_t p = s - (int64_t)(BT - 1) * DL - R;
                const auto& fin = acc[BT - 1][ROT ? 0 : pmod(k - (BT - 1) * DL - R, P)];
                auto put = [&](T* op) {
#pragma unroll
                    for (int yy = 0; yy < VY; ++yy) {
                        T c[VX];
                        LN::to_cells(c, fin[yy]);
#pragma unroll
                        for (int j = 0; j < NSG; ++j) {
                            if ((st_full >> (yy * NSG + j)) & 1u) {
                                if constexpr (K::XPAIR)
                                    *reinterpret_cast<float2*>(op + yy * a.py + j * SG) = make_float2(c[j * SG], c[j * SG + 1]);
                                else
                                    st_vec_global<T>(op + yy * a.py + j * SG, c + j * SG);
                            }
                            if constexpr (EDGE) {
#pragma unroll
                                for (int e = 0; e < SG; ++e)
                                    if ((st_elem >> (yy * VX + j * SG + e)) & 1u) op[yy * a.py + j * SG + e] = c[j * SG + e];
                            }
                        }
                    }
                };
                put(dst + st_off);
                // fused halo exchange: the neighbours' ghost planes, stored straight into their
                // (peer-mapped) buffers by the same thread (NEXT N1)
#ifndef AN5D_NO_PEER3D
                if constexpr (EDGE) {   // units reaching the send bands run the EDGE copy (kernel entry)
                    if (a.peer_lo && p < a.send_lo_end) put(static_cast<T*>(a.peer_lo) + (st_off + a.peer_lo_shift));
                    if (a.peer_hi && p >= a.send_hi_begin) put(static_cast<T*>(a.peer_hi) + (st_off + a.peer_hi_shift));
                }
#endif
#pragma unroll
                for (int yy = 0; yy < VY; ++yy) {
                    if (a.wc) {
                        const int y = gy0 + yy;
#pragma unroll
                        for (int xx = 0; xx < VX; ++xx) {
                            const int x = gx0 + xx;
                            if (y >= g.cy0 && y < g.cy1 && x >= g.cx0 && x < g.cx1)
                                atomicAdd(a.wc + (p * a.Ey + y) * (int64_t)a.Ex + x, 1);
                        }
                    }
                }
            }
            st_off += a.pz;
            if constexpr (ROT) {
                // slot j <- slot j+1: slot 0 (just completed and consumed) is recycled as the last
#pragma unroll
                for (int l = 0; l < BT; ++l)
#pragma unroll
                    for (int j = 0; j + 1 < P; ++j)
#pragma unroll
                        for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                            for (int e = 0; e < NE; ++e) acc[l][j][yy][e] = acc[l][j + 1][yy][e];
                if constexpr (RLOOP) {   // the recycled slot accumulates from zero (no first-tap multiply)
#pragma unroll
                    for (int l = 0; l < BT; ++l)
#pragma unroll
                        for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                            for (int e = 0; e < NE; ++e) acc[l][P - 1][yy][e] = E{};
                }
            }
        });
    }
    // drain: the PF planes still in flight must land before the block's shared memory is released
#pragma unroll
    for (int d = 0; d < PF; ++d) {
        wait_plane(slot_i);
        if (++slot_i == D) slot_i = 0;
    }
    // cluster: no block may exit (releasing its shared memory) while a neighbour can still read it
    if constexpr (CSPLIT) cluster_wait();
    else if constexpr (CFULL) cluster_sync_all();
}

// resident blocks per SM the register budget is shaped for: small fp32 patches (VY <= 2) fit two
// 256-thread blocks (<= 128 registers/thread), so one block's barrier and latency stalls overlap
// the other's; fp64 (twice the registers per cell) and high-order box keep one block and up to 255
// registers; 512-thread layouts one block at <= 128 registers (build.py / regcaps.json lower the
// cap with AN5D_MINB_CAP where ptxas reports spills)
template <typename T, int VY, int R, bool BOX, int TXT> constexpr int min_blocks_3d() {
    constexpr int m = (TXT == 16 && sizeof(T) == 4 && VY <= 2 && !(BOX && R >= 2)) ? 2 : 1;
#ifdef AN5D_MINB_CAP
    return m < AN5D_MINB_CAP ? m : AN5D_MINB_CAP;
#else
    return m;
#endif
}

// CL > 1: launched with cluster dimension (CL, 1, 1); the CL consecutive blocks of a cluster take
// the same unit (a cluster tile of CL x kTY rows) and block rank c its rows [c kTY, (c+1) kTY).
template <typename T, int R, int BT, int VY, bool BOX, int TXT = 16, int VX = 4, int CL = 1, int OS = 0>
__global__ void __launch_bounds__(TXT * 16, min_blocks_3d<T, VY, R, BOX, TXT>())
an5d_sweep3d(const Sweep3DArgs a, const __grid_constant__ Coeffs3D<T, R> cf, const __grid_constant__ CUtensorMap tmap) {
    using K = Kernel3DTraits<T, R, BT, VY, TXT, VX, OS>;
    pdl_wait();      // the previous sweep has completed (common.cuh PDL)
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* const smem = reinterpret_cast<T*>(smem_raw) + K::lead(CL);
    const int64_t unit = blockIdx.x / CL;
    const unsigned crank = CL > 1 ? cluster_ctarank() : 0;
    if (unit >= a.n_units) return;   // the whole cluster (same unit) leaves together
    int ty, tx;
    int64_t sb, sb_end;
    if (a.runs) {
        // run table (host-built, launch_sweep): consecutive stream blocks [sb, sb_end) of one tile in
        // one pass; blocks are dispatched in index order, so the table's order is the schedule
        const int4 r = a.runs[unit];
        ty = r.x;
        tx = r.y;
        sb = r.z;
        sb_end = r.w;
    } else {
        unit_to_tile3d(a, unit, ty, tx, sb);
        sb_end = sb + 1;
    }
    Unit3D g;
    {   // compute rows of the (cluster) tile, then this block's window and its share of them
        const int cy0 = R + ty * a.Cy, cy1 = min(cy0 + a.Cy, a.Ey - R);
        g.wy0 = cy0 - a.Hy + (int)crank * K::kTY;
        g.cy0 = max(cy0, g.wy0);
        g.cy1 = min(cy1, g.wy0 + K::kTYL);  // may be empty (a block below the array end)
    }
    g.cx0 = R + tx * a.Cx;
    g.cx1 = min(g.cx0 + a.Cx, a.Ex - R);
    g.wx0 = g.cx0 - a.Hx;
    g.p0 = a.out_lo + sb * a.h;
    g.p1 = min(a.out_lo + sb_end * a.h, a.out_hi);
    g.s_first = g.p0 - (int64_t)BT * R;
    g.s_end = g.p1 + (int64_t)BT * R;
    g.s_a = max(g.s_first, (int64_t)0);
    g.s_b = min(g.s_end, a.Ez);
    g.ring_xy = g.wy0 < R || g.wy0 + K::kTYL > a.Ey - R || g.wx0 < R || g.wx0 + K::kTXW > a.Ex - R;
    // z-ring planes and the array's z ends are handled by both variants (uniform per-step checks);
    // the EDGE variant is only for tiles whose window touches the x/y ring or the array end
    if (threadIdx.x == 0) tma_prefetch_desc(&tmap);
    // units storing planes of the fused-exchange send bands run the EDGE copy too
    if (g.ring_xy || (a.peer_lo && g.p0 < a.send_lo_end) || (a.peer_hi && g.p1 > a.send_hi_begin))
        sweep3d_unit<T, R, BT, VY, BOX, true, TXT, VX, CL, OS>(a, cf, smem, g, &tmap, crank);
    else sweep3d_unit<T, R, BT, VY, BOX, false, TXT, VX, CL, OS>(a, cf, smem, g, &tmap, crank);
}

}  // namespace an5d
