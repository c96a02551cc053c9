"""Pins of the multi-field system oracle (NEXT N4) against values fixed by mathematics.

  A_i' = sum_j sum_d c[i, j][d] A_j[x + d]      (every statement reads the previous step)

* decoupled blocks reduce to independent runs of the single-field oracle (itself pinned in
  test_oracle_pins.py) -- bit for bit;
* constant states evolve by the 2x2 matrix of block sums, M^T (closed form);
* a single-step impulse in field j shows the MIRRORED block (i, j) in field i (catches a
  transposed block index or an unmirrored offset);
* the T-step impulse response equals the T-fold block convolution (scipy.signal.convolve),
  exact on integer tables;
* the ring is never written; the thread count does not change a bit.
"""
import numpy as np
import pytest
from scipy import signal

import inputs
import oracle


@pytest.mark.parametrize("shape", [inputs.STAR, inputs.BOX])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_decoupled_equals_single_field_runs(shape, dtype):
    ndim, rad, nf = 2, 2, 2
    tab = inputs.system_table(ndim, rad, shape, nf, seed=4)
    tab[0, 1] = 0
    tab[1, 0] = 0
    f = inputs.system_fields(9, nf, (21, 26))
    out = oracle.run_system(f, rad, shape, tab, 6, dtype)
    for i in range(nf):
        assert np.array_equal(out[i], oracle.run(f[i], rad, shape, tab[i, i], 1.0, 6, dtype))


@pytest.mark.parametrize("shape", [inputs.STAR, inputs.BOX])
def test_constant_state_matrix_power(shape):
    """Fields constant at (a_0, ..., a_{n-1}): every statement sees constants, so the state moves by
    M = block sums, a_T = M^T a_0, at every cell farther than T rad from the ring."""
    ndim, rad, nf, T = 2, 1, 2, 5
    tab = inputs.system_table(ndim, rad, shape, nf, seed=6)
    M = tab.reshape(nf, nf, -1).sum(-1)
    a0 = np.array([0.25, 0.75])
    f = np.stack([np.full((19, 23), v) for v in a0])
    out = oracle.run_system(f, rad, shape, tab, T, np.float64)
    aT = np.linalg.matrix_power(M, T) @ a0
    y, x = np.indices((19, 23))
    far = np.minimum.reduce([y, x, 18 - y, 22 - x]) > T * rad
    for i in range(nf):
        assert np.max(np.abs(out[i][far] - aT[i])) <= 1e-15
    # row sums are 1 (dyadic tables): equal constants are an exact fixed point everywhere
    f1 = np.full((nf, 19, 23), 0.375)
    assert np.array_equal(oracle.run_system(f1, rad, shape, tab, T, np.float64), f1)


@pytest.mark.parametrize("ndim,shape", [(2, inputs.STAR), (2, inputs.BOX), (3, inputs.STAR)])
def test_impulse_shows_mirrored_block(ndim, shape):
    rad, nf = 2, 2
    tab = inputs.system_table(ndim, rad, shape, nf, seed=8)
    n = 11
    ext = (n,) * ndim
    x0 = (n // 2,) * ndim
    w = 2 * rad + 1
    for j in range(nf):
        f = np.zeros((nf,) + ext)
        f[(j,) + x0] = 1.0
        out = oracle.run_system(f, rad, shape, tab, 1, np.float64)
        win = tuple(slice(c - rad, c + rad + 1) for c in x0)
        for i in range(nf):
            mirrored = tab[i, j][tuple(slice(None, None, -1) for _ in range(ndim))]
            assert np.array_equal(out[i][win], mirrored), (i, j)
            rest = out[i].copy()
            rest[win] = 0
            assert not rest.any()
        assert w == 2 * rad + 1


def test_T_step_impulse_block_convolution():
    """Integer +-1 tables: the response to a unit impulse after T steps is the T-fold block
    convolution R_i^(t+1) = sum_j K_ij * R_j^(t) with K_ij the mirrored block -- exact in fp64."""
    ndim, rad, shape, nf, T = 2, 1, inputs.BOX, 2, 4
    tab = inputs.system_table(ndim, rad, shape, nf, seed=10, kind="pm1")
    n = 2 * T * rad + 2 * rad + 7
    x0 = (n // 2, n // 2)
    f = np.zeros((nf, n, n))
    f[(0,) + x0] = 1.0
    out = oracle.run_system(f, rad, shape, tab, T, np.float64)
    R = [np.ones((1, 1)), np.zeros((1, 1))]
    for _ in range(T):
        R = [sum(signal.convolve(R[j], tab[i, j][::-1, ::-1], mode="full") for j in range(nf)) for i in range(nf)]
    h = T * rad
    for i in range(nf):
        got = out[i][x0[0] - h:x0[0] + h + 1, x0[1] - h:x0[1] + h + 1]
        assert np.array_equal(got, np.asarray(R[i])), i


def test_ring_and_threads():
    tab = inputs.system_table(2, 1, inputs.STAR, 2, seed=12)
    f = inputs.system_fields(3, 2, (30, 41))
    a = oracle.run_system(f, 1, inputs.STAR, tab, 7, np.float32, nthreads=1)
    b = oracle.run_system(f, 1, inputs.STAR, tab, 7, np.float32, nthreads=4)
    assert np.array_equal(a, b)
    ring = np.ones((30, 41), bool)
    ring[1:-1, 1:-1] = False
    for i in range(2):
        assert np.array_equal(a[i][ring], f[i].astype(np.float32)[ring])
    assert np.array_equal(oracle.run_system(f, 1, inputs.STAR, tab, 0, np.float64), f)
