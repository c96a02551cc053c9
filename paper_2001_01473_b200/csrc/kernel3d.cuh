// kernel3d.cuh -- N.5D (2.5D spatial + b_T temporal) blocked 3D stencil sweep for sm_100a.
//
// PAPER.md mapping (AN5D, arXiv 2001.01473):
//   * a thread block owns a (y, x) tile of b_Sy x b_Sx cells and streams along z, the outermost
//     dimension (2.5D blocking);
//   * b_T computational streams; level T works on plane s - T*rad (fig:tier);
//   * overlapped tiles with b_T*rad halos recomputed redundantly, compute region stored
//     (P:166-172);
//   * in-plane neighbours are exchanged through a DOUBLE-BUFFERED shared-memory plane, one block
//     barrier per level (Table 1 "2 x n_thr x n_word");
//   * stream-dimension neighbours never touch shared memory: every arriving plane of level T-1
//     updates the 2*rad+1 in-flight output planes of level T held in registers (associative partial
//     sums; for star the off-centre planes add one tap);
//   * fixed register slots indexed by plane mod (2*rad+1), loop unrolled by that period;
//     for box stencils with rad >= 2 (>= 125 taps per cell) the code size of that unroll is not
//     worth it: the slots are rotated instead (2*rad moves per cell against (2rad+1)^3 FMAs);
//   * the boundary ring is never computed: ring planes / cells are re-read from the sweep input
//     whenever a level needs them.
//
// B200 design:
//   * 256 threads, 16 x 16; each thread owns a VY x 4 patch of cells (register tiling: 4 x-cells =
//     one 16-byte vector for fp32, two for fp64), so a plane of the tile is 64 x (16*VY) cells;
//   * the streamed level-0 plane is staged by cp.async (LDGSTS, 16 bytes per request) into a ring
//     of D shared-memory planes, D-1 planes ahead of the computation: no registers are spent on
//     prefetch and HBM latency is covered by the pipeline depth, not by occupancy;
//   * level 1 reads its own patch + halo straight from the staged plane (no extra store);
//     levels >= 2 store their patch into the double-buffered exchange plane.
#pragma once
#include "common.cuh"

namespace an5d {

struct Sweep3DArgs {
    const void* src;
    void* dst;
    int64_t pz, py;          // plane and row strides (elements)
    int64_t Ez;              // local planes
    int64_t g_off, gEz;      // global index of local plane 0, global z extent (slab mode)
    int64_t out_lo, out_hi;  // local output planes [out_lo, out_hi)
    int64_t h;               // stream-block length
    int64_t n_units;         // units handled by this launch
    int64_t n_sb, sb_lo, sb_hi;
    int32_t* wc;             // debug store counts (dense Ez x Ey x Ex) or nullptr
    int Ey, Ex;
    int Cy, Cx;              // compute region per tile
    int Hy, Hx;              // loaded halo per side (Hy = degree*rad; Hx rounded to 16 bytes)
    int nty, ntx;            // tiles along y, x
    int ty_lo, ty_hi, tx_lo, tx_hi;  // interior box in tile space
};

template <typename T, int R, int VY>
struct Kernel3DTraits {
    static constexpr int A = VecOf<T>::A;
    static constexpr int VX = 4;
    static constexpr int TXT = 16, TYT = 16;
    static constexpr int kThreads = TXT * TYT;
    static constexpr int kTX = TXT * VX, kTY = TYT * VY;
    static constexpr int XP = 4;                  // x padding of the smem planes (>= rad, 16B)
    static constexpr int TXP = kTX + 2 * XP;
    static constexpr int TYP = kTY + 2 * R;
    static constexpr int PLANE = TYP * TXP;       // elements per smem plane
    static constexpr int D = 3;                   // staged level-0 planes (prefetch depth D-1)
    static constexpr size_t kSmemBytes = (size_t)(D + 2) * PLANE * sizeof(T);
};

// Complement of the rectangle [r_lo, r_hi) x [c_lo, c_hi) in an nrows x ncols grid.
__device__ __forceinline__ void frame2d(int64_t u, int nrows, int ncols, int r_lo, int r_hi, int c_lo,
                                        int c_hi, int& row, int& col) {
    const int64_t n_bot = (int64_t)r_lo * ncols;
    if (u < n_bot) { row = (int)(u / ncols); col = (int)(u % ncols); return; }
    u -= n_bot;
    const int64_t n_top = (int64_t)(nrows - r_hi) * ncols;
    if (u < n_top) { row = r_hi + (int)(u / ncols); col = (int)(u % ncols); return; }
    u -= n_top;
    const int w = c_lo + (ncols - c_hi);
    row = r_lo + (int)(u / w);
    const int i = (int)(u % w);
    col = i < c_lo ? i : c_hi + (i - c_lo);
}

template <bool EDGE>
__device__ __forceinline__ void unit_to_tile3d(const Sweep3DArgs& a, int64_t u, int& ty, int& tx,
                                               int64_t& sb) {
    if constexpr (!EDGE) {
        const int nix = a.tx_hi - a.tx_lo, niy = a.ty_hi - a.ty_lo;
        tx = a.tx_lo + (int)(u % nix);
        ty = a.ty_lo + (int)((u / nix) % niy);
        sb = a.sb_lo + u / ((int64_t)nix * niy);
    } else {
        const int64_t NT = (int64_t)a.nty * a.ntx;
        const int64_t n_bot = a.sb_lo * NT;
        if (u < n_bot) { sb = u / NT; const int t = (int)(u % NT); ty = t / a.ntx; tx = t % a.ntx; return; }
        u -= n_bot;
        const int64_t n_top = (a.n_sb - a.sb_hi) * NT;
        if (u < n_top) {
            sb = a.sb_hi + u / NT; const int t = (int)(u % NT); ty = t / a.ntx; tx = t % a.ntx; return;
        }
        u -= n_top;
        const int64_t F = NT - (int64_t)(a.ty_hi - a.ty_lo) * (a.tx_hi - a.tx_lo);
        sb = a.sb_lo + u / F;
        frame2d(u % F, a.nty, a.ntx, a.ty_lo, a.ty_hi, a.tx_lo, a.tx_hi, ty, tx);
    }
}

template <typename T, int R, int BT, int VY, bool BOX, bool EDGE>
__global__ void __launch_bounds__(256, 1)
an5d_sweep3d(const Sweep3DArgs a, const Coeffs<T, (2 * R + 1) * (2 * R + 1) * (2 * R + 1)> cf) {
    using K = Kernel3DTraits<T, R, VY>;
    constexpr int A = K::A, VX = K::VX, TXP = K::TXP, XP = K::XP, D = K::D;
    constexpr int P = 2 * R + 1, W = 2 * R + 1;
    constexpr int NCH = VX / A;
    constexpr bool ROT = BOX && R >= 2;           // rotate slots instead of unrolling by P
    constexpr int U = ROT ? 1 : P;                // unroll factor of the stream loop
    static_assert(R <= XP, "x padding must cover the radius");

    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* const smem = reinterpret_cast<T*>(smem_raw);

    const int64_t unit = blockIdx.x;
    if (unit >= a.n_units) return;
    int tile_y, tile_x;
    int64_t sb;
    unit_to_tile3d<EDGE>(a, unit, tile_y, tile_x, sb);

    const T* __restrict__ src = static_cast<const T*>(a.src);
    T* __restrict__ dst = static_cast<T*>(a.dst);

    const int tid = threadIdx.x;
    const int txi = tid % K::TXT, tyi = tid / K::TXT;
    const int xs = txi * VX, ys = tyi * VY;                 // patch origin in the tile window

    const int cy0 = R + tile_y * a.Cy, cy1 = min(cy0 + a.Cy, a.Ey - R);
    const int cx0 = R + tile_x * a.Cx, cx1 = min(cx0 + a.Cx, a.Ex - R);
    const int wy0 = cy0 - a.Hy, wx0 = cx0 - a.Hx;          // loaded window origin
    const int gy0 = wy0 + ys, gx0 = wx0 + xs;               // this thread's first cell
    const int64_t p0 = a.out_lo + sb * a.h;
    const int64_t p1 = min(p0 + a.h, a.out_hi);
    const int64_t s_first = p0 - (int64_t)BT * R;
    const int64_t s_end = p1 + (int64_t)BT * R;

    // smem plane element offset of this thread's patch origin
    const int own = (ys + R) * TXP + (xs + XP);
    T* const stage = smem;                                   // D staged level-0 planes
    T* const xbuf = smem + D * K::PLANE;                     // 2 exchange planes

    // per-thread masks (EDGE only): ring cells and store coverage
    uint32_t ring_mask = 0;
    if constexpr (EDGE) {
#pragma unroll
        for (int yy = 0; yy < VY; ++yy)
#pragma unroll
            for (int xx = 0; xx < VX; ++xx) {
                const int y = gy0 + yy, x = gx0 + xx;
                const bool in = y >= 0 && y < a.Ey && x >= 0 && x < a.Ex;
                const bool ring = y < R || y >= a.Ey - R || x < R || x >= a.Ex - R;
                if (in && ring) ring_mask |= 1u << (yy * VX + xx);
            }
    }

    // ---- level-0 staging: cp.async of this thread's patch rows of plane q into stage slot -----
    auto stage_plane = [&](int64_t q, T* slot) {
        if constexpr (!EDGE) {
            if (q < s_end) {
                const T* gp = src + q * a.pz + (int64_t)gy0 * a.py + gx0;
#pragma unroll
                for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                    for (int j = 0; j < NCH; ++j)
                        cp_async16(slot + own + yy * TXP + j * A, gp + yy * a.py + j * A, 16);
            }
        } else {
            if (q >= 0 && q < a.Ez && q < s_end) {
                const T* gp = src + q * a.pz;
#pragma unroll
                for (int yy = 0; yy < VY; ++yy) {
                    const int y = gy0 + yy;
#pragma unroll
                    for (int j = 0; j < NCH; ++j) {
                        const int x = gx0 + j * A;
                        T* sd = slot + own + yy * TXP + j * A;
                        if (y < 0 || y >= a.Ey || x >= a.Ex || x + A <= 0) {
                            cp_async16(sd, src, 0);                       // zero fill
                        } else if (x >= 0) {
                            const int nb = min(A, a.Ex - x) * (int)sizeof(T);
                            cp_async16(sd, gp + (int64_t)y * a.py + x, nb);
                        } else {                                          // straddles x = 0
#pragma unroll
                            for (int e = 0; e < A; ++e)
                                sd[e] = (x + e >= 0) ? gp[(int64_t)y * a.py + x + e] : T(0);
                        }
                    }
                }
            }
        }
        cp_async_commit();
    };

    // ---- register state --------------------------------------------------------------------------
    T acc[BT][P][VY][VX];
#pragma unroll
    for (int l = 0; l < BT; ++l)
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                for (int xx = 0; xx < VX; ++xx) acc[l][k][yy][xx] = T(0);

    const int64_t s_a = EDGE ? max(s_first, (int64_t)0) : s_first;
    const int64_t base0 = s_a - (s_a % U);
    // prologue: stage planes base0 .. base0 + D - 2
#pragma unroll
    for (int d = 0; d < D - 1; ++d) stage_plane(base0 + d, stage + (int)((base0 + d) % D) * K::PLANE);

    int xb = 0;  // exchange buffer parity
    for (int64_t base = base0; base < s_end; base += U) {
        static_for<0, U>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            const int64_t s = base + k;
            T* const cur = stage + (int)(s % D) * K::PLANE;
            cp_async_wait<D - 2>();
            __syncthreads();                                 // plane s visible; slot (s-1)%D free
            stage_plane(s + D - 1, stage + (int)((s + D - 1) % D) * K::PLANE);

            T u[VY][VX];
            static_for<1, BT + 1>([&](auto lc) {
                constexpr int L = decltype(lc)::value;
                const T* pl;
                if constexpr (L == 1) {
                    pl = cur;
#pragma unroll
                    for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                        for (int j = 0; j < NCH; ++j) ld_vec_shared<T>(&u[yy][j * A], pl + own + yy * TXP + j * A);
                } else {
                    if constexpr (EDGE) {
                        const int64_t q = s - (int64_t)(L - 1) * R;
                        const int64_t gq = q + a.g_off;
                        if (q < 0 || q >= a.Ez) {
#pragma unroll
                            for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                                for (int xx = 0; xx < VX; ++xx) u[yy][xx] = T(0);
                        } else if (gq < R || gq >= a.gEz - R) {
                            const T* gp = src + q * a.pz;
#pragma unroll
                            for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                                for (int xx = 0; xx < VX; ++xx) {
                                    const int y = gy0 + yy, x = gx0 + xx;
                                    u[yy][xx] = (y >= 0 && y < a.Ey && x >= 0 && x < a.Ex)
                                                    ? gp[(int64_t)y * a.py + x] : T(0);
                                }
                        } else if (ring_mask) {
                            const T* gp = src + q * a.pz;
#pragma unroll
                            for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                                for (int xx = 0; xx < VX; ++xx)
                                    if (ring_mask & (1u << (yy * VX + xx)))
                                        u[yy][xx] = gp[(int64_t)(gy0 + yy) * a.py + gx0 + xx];
                        }
                    }
                    T* xw = xbuf + xb * K::PLANE;
                    xb ^= 1;
#pragma unroll
                    for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                        for (int j = 0; j < NCH; ++j) st_vec_shared<T>(xw + own + yy * TXP + j * A, &u[yy][j * A]);
                    __syncthreads();
                    pl = xw;
                }
                // ---- gather the in-plane neighbourhood of the patch ------------------------------
                T uh[VY + 2 * R][VX + 2 * R];
#pragma unroll
                for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                    for (int xx = 0; xx < VX; ++xx) uh[R + yy][R + xx] = u[yy][xx];
#pragma unroll
                for (int yy = -R; yy < VY + R; ++yy) {
                    const bool own_row = yy >= 0 && yy < VY;
                    if (!own_row) {
#pragma unroll
                        for (int j = 0; j < NCH; ++j)
                            ld_vec_shared<T>(&uh[R + yy][R + j * A], pl + own + yy * TXP + j * A);
                    }
                    if (own_row || BOX) {
#pragma unroll
                        for (int r = 1; r <= R; ++r) {
                            uh[R + yy][R - r] = pl[own + yy * TXP - r];
                            uh[R + yy][R + VX - 1 + r] = pl[own + yy * TXP + VX - 1 + r];
                        }
                    }
                }
                // ---- contributions of the arriving plane q = s-(L-1)R to outputs p = q - dz ------
                static_for<0, 2 * R + 1>([&](auto dc) {
                    constexpr int dz = R - decltype(dc)::value;
                    constexpr int slot = ROT ? (R - dz) : pmod(k - (L - 1) * R - dz, P);
                    if constexpr (BOX) {
#pragma unroll
                        for (int dy = -R; dy <= R; ++dy)
#pragma unroll
                            for (int dx = -R; dx <= R; ++dx) {
                                const T c = cf.c[((dz + R) * W + (dy + R)) * W + (dx + R)];
#pragma unroll
                                for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                                    for (int xx = 0; xx < VX; ++xx) {
                                        T& o = acc[L - 1][slot][yy][xx];
                                        const T f = uh[R + yy + dy][R + xx + dx];
                                        if (dz == -R && dy == -R && dx == -R) o = c * f;
                                        else o = fma(c, f, o);
                                    }
                            }
                    } else if constexpr (dz != 0) {
                        const T c = cf.c[((dz + R) * W + R) * W + R];
#pragma unroll
                        for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                            for (int xx = 0; xx < VX; ++xx) {
                                T& o = acc[L - 1][slot][yy][xx];
                                if (dz == -R) o = c * u[yy][xx];
                                else o = fma(c, u[yy][xx], o);
                            }
                    } else {
                        // in-plane cross in lexicographic (dy, dx) order
#pragma unroll
                        for (int dy = -R; dy <= R; ++dy) {
#pragma unroll
                            for (int dx = -R; dx <= R; ++dx) {
                                if (dy != 0 && dx != 0) continue;
                                const T c = cf.c[(R * W + (dy + R)) * W + (dx + R)];
#pragma unroll
                                for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                                    for (int xx = 0; xx < VX; ++xx) {
                                        T& o = acc[L - 1][slot][yy][xx];
                                        o = fma(c, uh[R + yy + dy][R + xx + dx], o);
                                    }
                            }
                        }
                    }
                });
                constexpr int done = ROT ? 0 : pmod(k - (L - 1) * R - R, P);
#pragma unroll
                for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                    for (int xx = 0; xx < VX; ++xx) u[yy][xx] = acc[L - 1][done][yy][xx];
                if constexpr (ROT) {
#pragma unroll
                    for (int j = 0; j + 1 < P; ++j)
#pragma unroll
                        for (int yy = 0; yy < VY; ++yy)
#pragma unroll
                            for (int xx = 0; xx < VX; ++xx) acc[L - 1][j][yy][xx] = acc[L - 1][j + 1][yy][xx];
                }
            });
            // ---- STORE level BT plane p = s - BT*R, compute region only ----------------------------
            const int64_t p = s - (int64_t)BT * R;
            if (p >= p0 && p < p1) {
                T* op = dst + p * a.pz;
#pragma unroll
                for (int yy = 0; yy < VY; ++yy) {
                    const int y = gy0 + yy;
                    if (y < cy0 || y >= cy1) continue;
#pragma unroll
                    for (int j = 0; j < NCH; ++j) {
                        const int x = gx0 + j * A;
                        if (x >= cx0 && x + A <= cx1) {
                            st_vec_global<T>(op + (int64_t)y * a.py + x, &u[yy][j * A]);
                        } else if (EDGE && x + A > cx0 && x < cx1) {
#pragma unroll
                            for (int e = 0; e < A; ++e)
                                if (x + e >= cx0 && x + e < cx1) op[(int64_t)y * a.py + x + e] = u[yy][j * A + e];
                        }
                    }
                    if (a.wc) {
#pragma unroll
                        for (int xx = 0; xx < VX; ++xx) {
                            const int x = gx0 + xx;
                            if (x >= cx0 && x < cx1) atomicAdd(a.wc + (p * a.Ey + y) * (int64_t)a.Ex + x, 1);
                        }
                    }
                }
            }
        });
    }
    cp_async_wait<0>();
}

}  // namespace an5d
