"""Pins of the CPU oracle against values fixed by the paper and by mathematics (not by itself).

Each test names the property and where it comes from (SURVEY.md §8(c) "What pins each part",
BASELINE.json north_star "oracle is itself checked on invariants").  Chosen so that a dropped tap,
a sign/index error, a transposed table or a wrong boundary fails at least one of them.
"""
import itertools

import numpy as np
import pytest
from scipy import signal

import inputs
import oracle

CASES = [(2, 1, inputs.STAR), (2, 2, inputs.BOX), (2, 3, inputs.STAR), (3, 1, inputs.BOX), (3, 2, inputs.STAR),
         (3, 1, inputs.STAR), (2, 1, inputs.BOX)]


def _ext(ndim, rad, n):
    return (n + 2 * rad,) * ndim


@pytest.mark.parametrize("ndim,rad,shape", CASES)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_constant_field_fixed_point(ndim, rad, shape, dtype):
    """Constant field is preserved when sum(c) == 1 (north_star invariant 1); dyadic c => exact."""
    tab, div = inputs.coeff_table(ndim, rad, shape, seed=11)
    assert tab.sum() == 1.0
    g = np.full(_ext(ndim, rad, 9 if ndim == 3 else 17), 0.375)
    out = oracle.run(g, rad, shape, tab, div, T=7, dtype=dtype)
    assert np.array_equal(out, g.astype(dtype))


@pytest.mark.parametrize("ndim,rad,shape", CASES)
@pytest.mark.parametrize("axis", [0, -1])
def test_linear_field_fixed_point(ndim, rad, shape, axis):
    """A symmetric stencil (c_d = c_-d, sum 1) maps a linear field a + b x_i to itself exactly
    (north_star invariant 2): sum_d c_d (a + b (x + d_i)) = a + b x since sum_d c_d d_i = 0."""
    tab, div = inputs.coeff_table(ndim, rad, shape, seed=5, symmetric=True)
    n = 9 if ndim == 3 else 15
    ext = _ext(ndim, rad, n)
    idx = np.indices(ext)[axis].astype(np.float64)
    g = 0.5 + 0.0625 * idx
    for dtype in (np.float32, np.float64):
        out = oracle.run(g, rad, shape, tab, div, T=5, dtype=dtype)
        assert np.array_equal(out, g.astype(dtype))


def test_linear_field_asymmetric_drifts():
    """Control for the linear pin: an ASYMMETRIC table moves a linear field by b*sum_d c_d d_i per
    step (a sign error in the offsets would flip the drift)."""
    ndim, rad, shape = 2, 1, inputs.STAR
    tab, _ = inputs.coeff_table(ndim, rad, shape, seed=3)
    drift = sum(tab[d0 + rad, d1 + rad] * d1 for d0, d1 in itertools.product(range(-rad, rad + 1), repeat=2))
    assert drift != 0
    ext = _ext(ndim, rad, 31)
    x = np.indices(ext)[1].astype(np.float64)
    g = 0.25 + 0.0078125 * x
    T = 3
    out = oracle.run(g, rad, shape, tab, 1.0, T=T, dtype=np.float64)
    # cells farther than T*rad from the ring are pure: f + T * b * drift
    core = (slice(rad + T * rad, ext[0] - rad - T * rad),) * 2
    assert np.allclose(out[core], g[core] + T * 0.0078125 * drift, rtol=0, atol=1e-15)


@pytest.mark.parametrize("ndim,rad,shape", CASES)
def test_quadratic_field_closed_form(ndim, rad, shape):
    """f = sum_i a_i x_i^2: each step adds q = sum_d c_d sum_i a_i d_i^2 (SURVEY §8(c) pin (iii));
    after T steps f_T = f_0 + T q at every cell farther than T*rad from the ring.  Pins temporal
    composition (a step applied twice or skipped changes T q)."""
    tab, div = inputs.coeff_table(ndim, rad, shape, seed=7, symmetric=True)
    n = 13 if ndim == 3 else 25
    ext = _ext(ndim, rad, n)
    a = [0.25, 0.5, 0.125][:ndim]
    ix = np.indices(ext).astype(np.float64)
    g = sum(a[i] * ix[i] ** 2 for i in range(ndim))
    q = 0.0
    for d in itertools.product(range(-rad, rad + 1), repeat=ndim):
        c = tab[tuple(v + rad for v in d)]
        q += c * sum(a[i] * d[i] ** 2 for i in range(ndim))
    T = 3
    out = oracle.run(g, rad, shape, tab, div, T=T, dtype=np.float64)
    core = tuple(slice(rad + T * rad, e - rad - T * rad) for e in ext)
    assert np.array_equal(out[core], g[core] + T * q)


@pytest.mark.parametrize("ndim,rad,shape", CASES)
def test_single_step_impulse_is_mirrored_table(ndim, rad, shape):
    """delta at x0, T=1 => out(x0 - d) = c_d: the impulse response reproduces the coefficient table,
    mirrored (north_star invariant 3; identical to the table only for symmetric tables, so an
    asymmetric table is used -- an unmirrored reading fails)."""
    tab, div = inputs.coeff_table(ndim, rad, shape, seed=13)
    n = 4 * rad + 3
    ext = _ext(ndim, rad, n)
    g = np.zeros(ext)
    x0 = tuple(e // 2 for e in ext)
    g[x0] = 1.0
    out = oracle.run(g, rad, shape, tab, div, T=1, dtype=np.float64)
    win = tuple(slice(c - rad, c + rad + 1) for c in x0)
    resp = out[win]
    mirrored = tab[(slice(None, None, -1),) * ndim]
    assert np.array_equal(resp, mirrored)
    # and zero everywhere else
    rest = out.copy()
    rest[win] = 0
    assert not rest.any()


@pytest.mark.parametrize("ndim,rad,shape,T", [(2, 1, inputs.STAR, 4), (2, 2, inputs.BOX, 3), (3, 1, inputs.BOX, 3),
                                              (3, 2, inputs.STAR, 2), (2, 4, inputs.STAR, 2)])
def test_T_step_impulse_is_self_convolution(ndim, rad, shape, T):
    """T-step impulse response = T-fold self-convolution of the mirrored kernel (SURVEY pin (v)),
    computed independently by scipy.signal.convolve; small integer taps => exact in fp64."""
    tab, _ = inputs.coeff_table(ndim, rad, shape, seed=21, kind="small")
    ext = _ext(ndim, rad, 2 * T * rad + 5)
    g = np.zeros(ext)
    x0 = tuple(e // 2 for e in ext)
    g[x0] = 1.0
    out = oracle.run(g, rad, shape, tab, 1.0, T=T, dtype=np.float64)
    k = tab[(slice(None, None, -1),) * ndim]
    resp = np.ones((1,) * ndim)
    for _ in range(T):
        resp = signal.convolve(resp, k, method="direct")
    win = tuple(slice(c - T * rad, c + T * rad + 1) for c in x0)
    assert resp.max() < 2 ** 53
    assert np.array_equal(out[win], resp)


def _brute(g, rad, shape, tab, div, T, dtype):
    """Pure-Python loops (tiny grids): for every interior cell, sum over the tap set in
    lexicographic order, IEEE ops in `dtype` via numpy scalars."""
    ndim = g.ndim
    ext = g.shape
    cur = g.astype(dtype).copy()
    nxt = cur.copy()
    taps = [d for d in itertools.product(range(-rad, rad + 1), repeat=ndim)
            if shape == inputs.BOX or sum(v != 0 for v in d) <= 1]
    cs = [dtype(tab[tuple(v + rad for v in d)]) for d in taps]
    dv = dtype(div)
    for _ in range(T):
        for x in itertools.product(*[range(rad, e - rad) for e in ext]):
            acc = dtype(0)
            for d, c in zip(taps, cs):
                acc = dtype(acc + dtype(c * cur[tuple(a + b for a, b in zip(x, d))]))
            nxt[x] = acc / dv if div != 1.0 else acc
        cur, nxt = nxt, cur
    return cur


@pytest.mark.parametrize("ndim,rad,shape,n", [(2, 1, inputs.STAR, 9), (2, 2, inputs.BOX, 8), (3, 1, inputs.BOX, 5),
                                              (3, 2, inputs.STAR, 5), (2, 1, inputs.STAR, 4)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("div_kind", ["dyadic", "int"])
def test_brute_force_tiny(ndim, rad, shape, n, dtype, div_kind):
    """Brute force on tiny grids (north_star: '<= 16^3 grids match'), random inputs, j-stencil
    divisor included; bit-identical since both sum the same taps in the same order."""
    tab, div = inputs.coeff_table(ndim, rad, shape, seed=31, kind=div_kind)
    ext = _ext(ndim, rad, n)
    g = inputs.global_grid(77, ext)
    T = 3
    got = oracle.run(g, rad, shape, tab, div, T=T, dtype=dtype)
    exp = _brute(g, rad, shape, tab, div, T, dtype)
    assert np.array_equal(got, exp)


def test_identity_and_uniform_examples():
    """identity stencil preserves the field; a uniform field maps to v * sum(c) / c_0."""
    ndim, rad = 2, 1
    g = inputs.global_grid(5, (10, 12))
    ident = np.zeros((3, 3))
    ident[1, 1] = 1.0
    assert np.array_equal(oracle.run(g, rad, inputs.STAR, ident, 1.0, 9, np.float64), g)
    tab = np.array([[0, 1, 0], [2, 3, 4], [0, 5, 0]], dtype=np.float64)
    u = np.full((7, 7), 2.0)
    out = oracle.run(u, rad, inputs.STAR, tab, 8.0, 1, np.float64)
    assert np.all(out[1:-1, 1:-1] == 2.0 * 15 / 8.0)
    assert np.all(out[0] == 2.0) and np.all(out[:, 0] == 2.0)   # ring untouched


def test_ring_never_written_and_T0():
    """Ring cells keep their input values (D1); T=0 returns the input."""
    tab, div = inputs.coeff_table(3, 2, inputs.BOX, seed=2)
    g = inputs.global_grid(9, (9, 10, 11))
    out = oracle.run(g, 2, inputs.BOX, tab, div, 4, np.float64)
    mask = np.ones(g.shape, bool)
    mask[2:-2, 2:-2, 2:-2] = False
    assert np.array_equal(out[mask], g[mask])
    assert not np.array_equal(out[~mask], g[~mask])
    assert np.array_equal(oracle.run(g, 2, inputs.BOX, tab, div, 0, np.float64), g)


def test_threads_do_not_change_result():
    """OpenMP partitioning of the outer loop must not change any bit (block order independence,
    S:469)."""
    tab, div = inputs.coeff_table(2, 1, inputs.BOX, seed=1)
    g = inputs.global_grid(3, (67, 45))
    a = oracle.run(g, 1, inputs.BOX, tab, div, 11, np.float32, nthreads=1)
    b = oracle.run(g, 1, inputs.BOX, tab, div, 11, np.float32, nthreads=3)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("ndim,rad,shape", [(2, 1, inputs.STAR), (2, 3, inputs.BOX), (3, 1, inputs.BOX),
                                            (3, 2, inputs.STAR)])
def test_steps_match_scipy_correlate_exact_integers(ndim, rad, shape):
    """An independent library routine as the reference: each time step is
    scipy.ndimage.correlate (out[x] = sum_d w[d] in[x + d], the definition of fig:jacobi2d /
    Table 2 with the ring held fixed), applied to the interior.  Integer taps and {-1, 0, 1}
    inputs keep every value an exact integer in fp64, so any summation order gives the same bits
    and the oracle must equal it exactly over several steps."""
    from scipy import ndimage
    tab, div = inputs.coeff_table(ndim, rad, shape, seed=12, kind="pm1")
    ext = tuple(9 + 2 * rad for _ in range(ndim))
    g = inputs.global_grid(3, ext, kind="pm")
    T = 3
    cur = g.copy()
    core = tuple(slice(rad, e - rad) for e in ext)
    for _ in range(T):
        nxt = cur.copy()
        nxt[core] = ndimage.correlate(cur, tab, mode="constant", cval=0.0)[core] / div
        cur = nxt
    got = oracle.run(g, rad, shape, tab, div, T, np.float64)
    assert np.abs(cur).max() < 2 ** 50
    assert np.array_equal(got, cur)
