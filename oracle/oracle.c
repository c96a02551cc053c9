/*
 * oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library.  The product path (paper_2001_01473_b200) never links, imports or calls it,
 * and it shares no source, header or helper with the CUDA path.
 *
 * What it computes: the plain double-buffered time loop of PAPER.md fig:jacobi2d,
 *   for t in 0..T-1:  A[(t+1)%2][x] = (sum_{d in taps} c_d * A[t%2][x+d]) / c_0   for interior x
 * with the stencil definitions of PAPER.md Table 2: star = centre plus +-k along one
 * axis at a time, box = the full (2 rad + 1)^N cube.  The constant ring of width rad
 * on every face is never written (fig:jacobi2d loop bounds 1..I_S).
 *
 * Readings:
 *   - C-8: arithmetic in the run's dtype, taps summed in canonical lexicographic order
 *     (d_outer, ..., d_x), separate multiply and add (built with -ffp-contract=off), true IEEE
 *     division by the divisor when divisor != 1 (the paper's fast-math reciprocal is NOT used here).
 *   - C-2 / C-3: coefficients are a run-time table (the paper's are compile-time constants);
 *     the divisor c_0 is a separate constant, not the centre tap.
 *   - Coefficients are rounded once, round-to-nearest, from double to the dtype.
 *   - The result of T steps is returned in `out` (T == 0 -> copy of the input).
 *
 * Layout: dense row-major, innermost x contiguous, extents INCLUDE the ring; ndim 1..3.
 * Parallelism: OpenMP over the outermost interior index (plain, untuned).
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Build the tap list (linear offsets + dtype-rounded coefficients) in lexicographic order of
 * the dense (2r+1)^ndim table; star keeps entries with at most one non-zero offset component. */
static int build_taps(int ndim, int rad, int shape, const double* coeffs, const int64_t* ext,
                      int64_t* lin_off, double* cval) {
    int w = 2 * rad + 1, n_dense = 1, n = 0;
    for (int i = 0; i < ndim; i++) n_dense *= w;
    for (int k = 0; k < n_dense; k++) {
        int d[3] = {0, 0, 0}, rem = k, nz = 0;
        for (int i = ndim - 1; i >= 0; i--) { d[i] = rem % w - rad; rem /= w; }
        for (int i = 0; i < ndim; i++) nz += (d[i] != 0);
        if (shape == 0 && nz > 1) continue; /* star: axis taps only */
        int64_t off = 0, stride = 1;
        for (int i = ndim - 1; i >= 0; i--) { off += d[i] * stride; stride *= ext[i]; }
        lin_off[n] = off;
        cval[n] = coeffs[k];
        n++;
    }
    return n;
}

#define DEFINE_ORACLE(NAME, T_)                                                                  \
int NAME(int ndim, int rad, int shape, const double* coeffs, double divisor,                     \
         const int64_t* ext, const T_* in, T_* out, int64_t T, int nthreads) {                   \
    if (ndim < 1 || ndim > 3 || rad < 1) return -1;                                              \
    int64_t ncell = 1;                                                                           \
    for (int i = 0; i < ndim; i++) { if (ext[i] < 2 * rad + 1) return -2; ncell *= ext[i]; }     \
    int w = 2 * rad + 1, n_dense = 1;                                                            \
    for (int i = 0; i < ndim; i++) n_dense *= w;                                                 \
    int64_t* lin_off = (int64_t*)malloc(sizeof(int64_t) * n_dense);                              \
    double* cd = (double*)malloc(sizeof(double) * n_dense);                                      \
    T_* c = (T_*)malloc(sizeof(T_) * n_dense);                                                   \
    int ntap = build_taps(ndim, rad, shape, coeffs, ext, lin_off, cd);                           \
    for (int k = 0; k < ntap; k++) c[k] = (T_)cd[k];                                             \
    const T_ div = (T_)divisor;                                                                  \
    const int use_div = (divisor != 1.0);                                                        \
    T_* a = (T_*)malloc(sizeof(T_) * ncell);                                                     \
    T_* b = (T_*)malloc(sizeof(T_) * ncell);                                                     \
    memcpy(a, in, sizeof(T_) * ncell);                                                           \
    memcpy(b, in, sizeof(T_) * ncell); /* ring of the second buffer = input ring */              \
    int64_t e0 = ndim >= 3 ? ext[ndim - 3] : 1;                                                  \
    int64_t e1 = ndim >= 2 ? ext[ndim - 2] : 1;                                                  \
    int64_t e2 = ext[ndim - 1];                                                                  \
    int64_t lo0 = ndim >= 3 ? rad : 0, hi0 = ndim >= 3 ? e0 - rad : 1;                          \
    int64_t lo1 = ndim >= 2 ? rad : 0, hi1 = ndim >= 2 ? e1 - rad : 1;                           \
    int64_t lo2 = rad, hi2 = e2 - rad;                                                           \
    for (int64_t t = 0; t < T; t++) {                                                            \
        const T_* src = a;                                                                       \
        T_* dst = b;                                                                             \
        int64_t nouter = (hi0 - lo0) * (hi1 - lo1);                                              \
        _Pragma("omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)")    \
        for (int64_t o = 0; o < nouter; o++) {                                                   \
            int64_t i0 = lo0 + o / (hi1 - lo1), i1 = lo1 + o % (hi1 - lo1);                      \
            int64_t rowbase = (i0 * e1 + i1) * e2;                                               \
            for (int64_t i2 = lo2; i2 < hi2; i2++) {                                             \
                int64_t x = rowbase + i2;                                                        \
                T_ acc = (T_)0;                                                                  \
                for (int k = 0; k < ntap; k++) {                                                 \
                    T_ prod = c[k] * src[x + lin_off[k]];                                        \
                    acc = acc + prod;                                                            \
                }                                                                                \
                dst[x] = use_div ? acc / div : acc;                                              \
            }                                                                                    \
        }                                                                                        \
        a = dst; b = (T_*)src;                                                                   \
    }                                                                                            \
    memcpy(out, a, sizeof(T_) * ncell);                                                          \
    free(a); free(b); free(lin_off); free(cd); free(c);                                          \
    return 0;                                                                                    \
}

DEFINE_ORACLE(oracle_run_f32, float)
DEFINE_ORACLE(oracle_run_f64, double)

/*
 * gradient2d (Table 2) -- the one non-linear benchmark:
 *   f'(x,y) = c * f(x,y) + 1.0 / sqrt(c_0 + sum_{i in {-1,+1}} ((f(x,y) - f(x+i,y))^2 + (f(x,y) - f(x,y+i))^2))
 * with c the centre coefficient and c_0 a constant (both run-time inputs; R-17).  Same
 * double-buffered loop, ring (rad = 1) never written, arithmetic in the run's dtype, evaluated
 * left to right as printed: the sum over i = -1 then i = +1, each term (x-difference squared) +
 * (y-difference squared); then c_0 + sum; IEEE sqrt and IEEE division (no FMA contraction).
 * Layout: dense row-major, 2D only, extents (E_y, E_x) include the ring.
 */
#define DEFINE_GRAD(NAME, T_, SQRT_)                                                             \
int NAME(double centre, double c0, const int64_t* ext, const T_* in, T_* out, int64_t T,         \
         int nthreads) {                                                                         \
    const int64_t ey = ext[0], ex = ext[1];                                                      \
    if (ey < 3 || ex < 3) return -2;                                                             \
    const T_ c = (T_)centre, k0 = (T_)c0;                                                        \
    T_* a = (T_*)malloc(sizeof(T_) * ey * ex);                                                   \
    T_* b = (T_*)malloc(sizeof(T_) * ey * ex);                                                   \
    memcpy(a, in, sizeof(T_) * ey * ex);                                                         \
    memcpy(b, in, sizeof(T_) * ey * ex);                                                         \
    for (int64_t t = 0; t < T; t++) {                                                            \
        const T_* src = a;                                                                       \
        T_* dst = b;                                                                             \
        _Pragma("omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)")    \
        for (int64_t y = 1; y < ey - 1; y++) {                                                   \
            for (int64_t x = 1; x < ex - 1; x++) {                                               \
                const T_ f = src[y * ex + x];                                                    \
                T_ sum = (T_)0;                                                                  \
                for (int i = -1; i <= 1; i += 2) {                                               \
                    const T_ dx = f - src[y * ex + (x + i)];                                     \
                    const T_ dy = f - src[(y + i) * ex + x];                                     \
                    const T_ sx = dx * dx, sy = dy * dy;                                         \
                    sum = sum + (sx + sy);                                                       \
                }                                                                                \
                const T_ cf = c * f;                                                             \
                dst[y * ex + x] = cf + (T_)1.0 / SQRT_(k0 + sum);                                \
            }                                                                                    \
        }                                                                                        \
        a = dst; b = (T_*)src;                                                                   \
    }                                                                                            \
    memcpy(out, a, sizeof(T_) * ey * ex);                                                        \
    free(a); free(b);                                                                            \
    return 0;                                                                                    \
}

DEFINE_GRAD(oracle_grad_f32, float, sqrtf)
DEFINE_GRAD(oracle_grad_f64, double, sqrt)

/*
 * Multi-field systems (NEXT N4, "multi-output temporal blocking to optimize multi-statement
 * stencils"): n_f arrays updated together, one statement per array, every statement
 * reading the previous time step of all arrays (Jacobi in time, like fig:jacobi2d P:406-413):
 *   for t in 0..T-1, for every field i, for every interior cell x:
 *       A_i[(t+1)%2][x] = sum_{j=0..n_f-1} sum_{d in taps} c_{ij,d} * A_j[t%2][x+d]
 * Table 2 shapes per (i, j) block (star or box), taps in lexicographic order, the j
 * sum outermost, in the run's dtype with separate multiply and add (built -ffp-contract=off).
 * Layout: fields are consecutive dense arrays (field f at f * prod(ext)); coeffs: n_f * n_f dense
 * (2r+1)^ndim tables, block (i, j) at (i * n_f + j) * (2r+1)^ndim (contribution of field j to
 * field i).  The ring of width rad of every field is never written.
 */
#define DEFINE_SYSTEM(NAME, T_)                                                                  \
int NAME(int ndim, int rad, int shape, int nf, const double* coeffs, const int64_t* ext,        \
         const T_* in, T_* out, int64_t T, int nthreads) {                                       \
    if (ndim < 1 || ndim > 3 || rad < 1 || nf < 1 || nf > 8) return -1;                         \
    int64_t ncell = 1;                                                                           \
    for (int i = 0; i < ndim; i++) { if (ext[i] < 2 * rad + 1) return -2; ncell *= ext[i]; }     \
    int w = 2 * rad + 1, n_dense = 1;                                                            \
    for (int i = 0; i < ndim; i++) n_dense *= w;                                                 \
    int64_t* lin_off = (int64_t*)malloc(sizeof(int64_t) * n_dense);                              \
    double* cd = (double*)malloc(sizeof(double) * n_dense);                                      \
    T_* c = (T_*)malloc(sizeof(T_) * n_dense * nf * nf);                                         \
    int ntap = 0;                                                                                \
    for (int b = 0; b < nf * nf; b++) {                                                          \
        ntap = build_taps(ndim, rad, shape, coeffs + (int64_t)b * n_dense, ext, lin_off, cd);    \
        for (int k = 0; k < ntap; k++) c[b * n_dense + k] = (T_)cd[k];                           \
    }                                                                                            \
    T_* a = (T_*)malloc(sizeof(T_) * ncell * nf);                                                \
    T_* bb = (T_*)malloc(sizeof(T_) * ncell * nf);                                               \
    memcpy(a, in, sizeof(T_) * ncell * nf);                                                      \
    memcpy(bb, in, sizeof(T_) * ncell * nf); /* rings of the second buffers = input rings */     \
    int64_t e0 = ndim >= 3 ? ext[ndim - 3] : 1;                                                  \
    int64_t e1 = ndim >= 2 ? ext[ndim - 2] : 1;                                                  \
    int64_t e2 = ext[ndim - 1];                                                                  \
    int64_t lo0 = ndim >= 3 ? rad : 0, hi0 = ndim >= 3 ? e0 - rad : 1;                          \
    int64_t lo1 = ndim >= 2 ? rad : 0, hi1 = ndim >= 2 ? e1 - rad : 1;                           \
    int64_t lo2 = rad, hi2 = e2 - rad;                                                           \
    for (int64_t t = 0; t < T; t++) {                                                            \
        const T_* src = a;                                                                       \
        T_* dst = bb;                                                                            \
        int64_t nouter = (hi0 - lo0) * (hi1 - lo1);                                              \
        for (int fi = 0; fi < nf; fi++) {                                                        \
            _Pragma("omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)") \
            for (int64_t o = 0; o < nouter; o++) {                                               \
                int64_t i0 = lo0 + o / (hi1 - lo1), i1 = lo1 + o % (hi1 - lo1);                  \
                int64_t rowbase = (i0 * e1 + i1) * e2;                                           \
                for (int64_t i2 = lo2; i2 < hi2; i2++) {                                         \
                    int64_t x = rowbase + i2;                                                    \
                    T_ acc = (T_)0;                                                              \
                    for (int fj = 0; fj < nf; fj++) {                                            \
                        const T_* s = src + (int64_t)fj * ncell;                                 \
                        const T_* cb = c + (int64_t)(fi * nf + fj) * n_dense;                    \
                        for (int k = 0; k < ntap; k++) {                                         \
                            T_ prod = cb[k] * s[x + lin_off[k]];                                 \
                            acc = acc + prod;                                                    \
                        }                                                                        \
                    }                                                                            \
                    dst[(int64_t)fi * ncell + x] = acc;                                          \
                }                                                                                \
            }                                                                                    \
        }                                                                                        \
        a = dst; bb = (T_*)src;                                                                  \
    }                                                                                            \
    memcpy(out, a, sizeof(T_) * ncell * nf);                                                     \
    free(a); free(bb); free(lin_off); free(cd); free(c);                                         \
    return 0;                                                                                    \
}

DEFINE_SYSTEM(oracle_system_f32, float)
DEFINE_SYSTEM(oracle_system_f64, double)

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
