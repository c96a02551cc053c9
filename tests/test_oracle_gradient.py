"""Pins of the gradient2d oracle (Table 2; NEXT N3) against closed forms.

  f'(x,y) = c f(x,y) + 1 / sqrt(c_0 + sum_{i=-1,+1} ((f - f(x+i,y))^2 + (f - f(x,y+i))^2))

None of these re-evaluates the oracle's per-cell expression: each uses a field for which the
gradient term has a closed form (constant: 0; linear a + b x + d y: 2 b^2 + 2 d^2; quadratic
q x^2: q^2 (8 x^2 + 2)), so a dropped neighbour, a one-sided sum, an axis mix-up, a missing
square, c and c_0 swapped or a missing reciprocal each fail one of them.
"""
import math

import numpy as np
import pytest

import oracle


def _dist_to_ring(shape):
    y, x = np.indices(shape)
    return np.minimum.reduce([y, x, shape[0] - 1 - y, shape[1] - 1 - x])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_constant_field_closed_form(dtype):
    """Constant field a: the gradient term vanishes, a_T = c^T a + k (1 - c^T) / (1 - c) with
    k = 1/sqrt(c_0), at every cell farther than T from the (unchanged) ring.  c = 1/2, c_0 = 1/4
    (k = 2) keep every value dyadic, so the closed form is exact in both precisions."""
    c, c0, a0 = 0.5, 0.25, 0.375
    g = np.full((23, 29), a0)
    for T in (1, 2, 5):
        out = oracle.run_gradient(g, c, c0, T, dtype)
        expect = c ** T * a0 + 2.0 * (1 - c ** T) / (1 - c)
        far = _dist_to_ring(g.shape) > T
        assert np.all(out[far] == dtype(expect)), T
        ring = _dist_to_ring(g.shape) == 0
        assert np.array_equal(out[ring], g.astype(dtype)[ring])


@pytest.mark.parametrize("axis", [0, 1])
def test_linear_field_one_step_exact(axis):
    """f = a + b u (u = x or y): the two neighbours along u differ by +-b, the other axis by 0, so
    f' = c f + 1/sqrt(c_0 + 2 b^2).  c_0 = 1/2, b = 1/2 gives sqrt(1) = 1: exact."""
    c, c0, a, b = 0.5, 0.5, 0.25, 0.5
    shape = (17, 21)
    u = np.indices(shape)[axis].astype(np.float64)
    g = a + b * u
    for dtype in (np.float32, np.float64):
        out = oracle.run_gradient(g, c, c0, 1, dtype)
        inner = _dist_to_ring(shape) >= 1
        assert np.array_equal(out[inner], (c * g + 1.0)[inner].astype(dtype))


@pytest.mark.parametrize("axis", [0, 1])
def test_linear_field_T_steps_recurrence(axis):
    """A linear field stays linear: slope b_{t+1} = c b_t, intercept a_{t+1} = c a_t + 1/sqrt(c_0 +
    2 b_t^2) -- the closed form of T steps at cells farther than T from the ring (fp64, to 1e-14)."""
    c, c0, a, b = 0.75, 0.3, 0.2, 0.4
    shape = (31, 27)
    u = np.indices(shape)[axis].astype(np.float64)
    g = a + b * u
    T = 6
    out = oracle.run_gradient(g, c, c0, T, np.float64)
    at, bt = a, b
    for _ in range(T):
        at, bt = c * at + 1.0 / math.sqrt(c0 + 2 * bt * bt), c * bt
    far = _dist_to_ring(shape) > T
    expect = at + bt * u
    assert np.max(np.abs(out[far] - expect[far])) <= 1e-14 * np.max(np.abs(expect[far]))


def test_plane_field_both_axes():
    """f = a + b x + d y with b != d: gradient term 2 b^2 + 2 d^2 (both axes, both sides).  A
    one-sided sum (b^2 + d^2), a single axis (2 b^2 or 2 d^2) or an axis swap of one difference
    (the cross terms) would change the value.  b = 1/4, d = 1/2, c_0 = 3/8: c_0 + 2b^2 + 2d^2 = 1."""
    c, c0, a, b, d = 0.5, 0.375, 0.125, 0.25, 0.5
    shape = (19, 25)
    y, x = np.indices(shape).astype(np.float64)
    g = a + b * x + d * y
    for dtype in (np.float32, np.float64):
        out = oracle.run_gradient(g, c, c0, 1, dtype)
        inner = _dist_to_ring(shape) >= 1
        assert np.array_equal(out[inner], (c * g + 1.0)[inner].astype(dtype))


def test_quadratic_field_one_step():
    """f = q x^2: (f - f(x+-1))^2 = q^2 (2x +- 1)^2, sum q^2 (8 x^2 + 2); y differences 0.
    f' = c q x^2 + 1/sqrt(c_0 + q^2 (8 x^2 + 2)) (fp64, to 4 ulp)."""
    c, c0, q = 0.625, 0.5, 0.03125
    shape = (9, 40)
    x = np.indices(shape)[1].astype(np.float64)
    g = q * x * x
    out = oracle.run_gradient(g, c, c0, 1, np.float64)
    expect = c * g + 1.0 / np.sqrt(c0 + q * q * (8 * x * x + 2))
    inner = _dist_to_ring(shape) >= 1
    assert np.max(np.abs(out[inner] - expect[inner]) / np.abs(expect[inner])) <= 4 * 2.0 ** -52


def test_single_cell_bump():
    """A single raised cell (height h) on a constant field: the cell itself sees 4 differences of
    h, each of its 4 axis neighbours one difference of -h, diagonal neighbours none (the
    gradient2d stencil is a 5-point star).  c_0 = 1/4, h = 1/2 -> sqrt(1/4 + 4/4) and
    sqrt(1/4 + 1/4) at the bump and its neighbours."""
    c, c0, base, h = 0.5, 0.25, 0.25, 0.5
    g = np.full((11, 13), base)
    g[5, 6] += h
    out = oracle.run_gradient(g, c, c0, 1, np.float64)
    assert out[5, 6] == c * (base + h) + 1.0 / math.sqrt(c0 + 4 * h * h)
    for (yy, xx) in ((4, 6), (6, 6), (5, 5), (5, 7)):
        assert out[yy, xx] == c * base + 1.0 / math.sqrt(c0 + h * h)
    for (yy, xx) in ((4, 5), (4, 7), (6, 5), (6, 7), (3, 6), (5, 8)):
        assert out[yy, xx] == c * base + 2.0


def test_T0_copy_and_thread_count():
    g = np.random.default_rng(3).random((40, 33))
    assert np.array_equal(oracle.run_gradient(g, 0.5, 1.0, 0, np.float64), g)
    a = oracle.run_gradient(g, 0.5, 1.0, 5, np.float32, nthreads=1)
    b = oracle.run_gradient(g, 0.5, 1.0, 5, np.float32, nthreads=4)
    assert np.array_equal(a, b)
