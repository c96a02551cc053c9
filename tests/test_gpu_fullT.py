"""Full-T parity (SURVEY.md §8(d) Policy; BASELINE.json north_star acceptance "after T steps").

* Every Table-2 stencil x {fp32, fp64} at the planner's choice of (b_T, vec) for the
  full BASELINE size (16384^2 / 512^3, T = 1000, the paper's protocol P:657-663), run for the full
  T = 1000 time steps on the reduced grids SURVEY.md allows (2048^2 / 128^3) and compared element
  by element with the oracle (relative L-inf <= 1e-5 fp32 / 1e-12 fp64, ring bit-exact).
* The headline workload (star2d1r fp32 16384^2, T = 1000) in bench.py's tuned configuration,
  compared with the oracle on the FULL grid, every cell.
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.float64: 1e-12}
NP = {torch.float32: np.float32, torch.float64: np.float64}

# interior size of the reduced grid (2D: n x n, 3D: n^3), T = 1000 (SURVEY.md §8(d) Policy sizes)
CASES = {name: (2048 if spec[0] == 2 else 128) for name, spec in inputs.BENCHMARKS.items()}


def rel_linf(got, exp, rad):
    core = tuple(slice(rad, e - rad) for e in exp.shape)
    den = np.abs(exp[core]).max()
    return np.abs(got[core].astype(np.float64) - exp[core].astype(np.float64)).max() / max(den, 1e-300)


def ring_equal(got, exp, rad):
    mask = np.ones(exp.shape, bool)
    mask[tuple(slice(rad, e - rad) for e in exp.shape)] = False
    return np.array_equal(got[mask], exp[mask])


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_full_T_parity_planner_config(an5d, name, dtype):
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    n, T = CASES[name], 1000
    interior = (n,) * ndim
    ext = tuple(v + 2 * rad for v in interior)
    full = (16384 + 2 * rad,) * 2 if ndim == 2 else (512 + 2 * rad,) * 3
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    pick = st.plan_config(full, 1000)                       # the planner's (b_T, vec) at BASELINE size
    cfg = st.plan_config(ext, T, {"bT": pick["bT"], "vec": pick["vec"], "n_thr": pick["n_thr"],
                                  "bS": pick["bS"]})                       # same layout; h for this grid
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_grid(ext, rad, dtype)
    b.fill_(float("nan"))
    st.run(a, b, T, cfg)
    torch.cuda.synchronize()
    got = b.cpu().numpy()
    exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
    assert ring_equal(got, exp, rad), (name, cfg)
    err = rel_linf(got, exp, rad)
    assert err <= TOL[dtype], (name, cfg, T, err)
    if shape == inputs.GRAD:   # individually rounded ops in the oracle's order: bit-identical
        assert np.array_equal(got, exp), (name, cfg, err)


@pytest.mark.slow
def test_full_size_headline_full_grid(an5d):
    name, n, T = "star2d1r", 16384, 1000
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = (n + 2 * rad,) * 2
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext).astype(np.float32)
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    a = an5d.to_grid(torch.from_numpy(g).cuda(), rad)
    b = an5d.empty_grid(ext, rad, torch.float32)
    cfg = st.tune(a, b, T, None, top_k=5)                   # bench.py's launch configuration
    cfg.pop("seconds_per_cell_step", None)
    a = an5d.to_grid(torch.from_numpy(g).cuda(), rad)
    b.fill_(float("nan"))
    st.run(a, b, T, cfg)
    torch.cuda.synchronize()
    got = b.cpu().numpy()
    del a, b
    exp = oracle.run(g, rad, shape, tab, div, T, np.float32)   # ~2.5 min on 16 host threads
    assert ring_equal(got, exp, rad), cfg
    err = rel_linf(got, exp, rad)
    assert err <= 1e-5, (err, cfg)
