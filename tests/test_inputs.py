"""The seeded input generators (module `inputs`, shared by oracle and GPU path; no stencil math)."""
import numpy as np
import torch

import inputs


def test_uniform24_range_and_exactness():
    v = inputs.uniform24(inputs.DEFAULT_SEED, np.arange(100000))
    assert v.min() >= 0.0 and v.max() < 1.0
    assert np.array_equal(v.astype(np.float32).astype(np.float64), v)   # exact in fp32
    assert np.array_equal(np.round(v * 2 ** 24), v * 2 ** 24)           # 24-bit grid
    assert abs(v.mean() - 0.5) < 0.01


def test_grid_is_function_of_global_index():
    """Slabs of the global grid see identical values (decomposition independence)."""
    ext = (12, 7, 9)
    full = inputs.global_grid(42, ext)
    part = inputs.global_grid(42, (5, 7, 9), outer_offset=4, outer_count=5, global_extents=ext)
    assert np.array_equal(full[4:9], part)


def test_torch_generator_matches_numpy():
    idx = np.arange(0, 1 << 20, 977, dtype=np.int64)
    idx = np.concatenate([idx, np.array([(1 << 33) + 5, (1 << 40) + 123])])
    a = inputs.uniform24(inputs.DEFAULT_SEED, idx)
    b = inputs.uniform24_torch(inputs.DEFAULT_SEED, torch.from_numpy(idx)).numpy()
    assert np.array_equal(a, b)


def test_coeff_tables():
    for name, (ndim, rad, shape, has_div) in inputs.BENCHMARKS.items():
        if shape == inputs.GRAD:   # centre c and c_0 only (test_benchmark_catalogue_matches_table2)
            continue
        _, _, _, tab, div = inputs.benchmark_problem(name)
        assert tab.shape == (2 * rad + 1,) * ndim
        nz = np.count_nonzero(tab)
        exp = (2 * rad + 1) ** ndim if shape == inputs.BOX else 2 * ndim * rad + 1
        assert nz == exp, name
        if has_div:
            assert div == tab.sum() and np.all(tab == np.round(tab))
        else:
            assert div == 1.0 and tab.sum() == 1.0    # dyadic, exact
            assert np.array_equal(tab.astype(np.float32).astype(np.float64), tab)
    sym, _ = inputs.coeff_table(3, 2, inputs.BOX, 9, symmetric=True)
    assert np.array_equal(sym, sym[::-1, ::-1, ::-1])


def test_benchmark_catalogue_matches_table2():
    """PAPER.md Table 2 benchmark list."""
    names = set(inputs.BENCHMARKS)
    for r in range(1, 5):
        for s in ("star2d", "box2d", "star3d", "box3d"):
            assert f"{s}{r}r" in names
    assert {"j2d5pt", "j2d9pt", "j3d27pt", "j2d9pt-gol"} <= names
    assert inputs.BENCHMARKS["j2d9pt-gol"] == (2, 1, inputs.BOX, True)   # 3x3 box / c_0
    assert inputs.BENCHMARKS["j2d9pt"][1] == 2   # "2nd-order"
    assert inputs.BENCHMARKS["gradient2d"] == (2, 1, inputs.GRAD, True)
    ndim, rad, shape, tab, c0 = inputs.benchmark_problem("gradient2d")
    assert tab.shape == (3, 3) and np.count_nonzero(tab) == 1 and 0 < tab[1, 1] < 1 and c0 >= 1
