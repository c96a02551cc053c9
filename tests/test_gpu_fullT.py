"""Full-T parity (SURVEY.md §8(d) Policy; BASELINE.json north_star acceptance "after T steps").

* Every Table-2 stencil x {fp32, fp64} at the planner's choice of (b_T, vec) for the
  full BASELINE size (16384^2 / 512^3, T = 1000, the paper's protocol P:657-663), run for the full
  T = 1000 time steps on a reduced grid (2048^2 ... 640^2, 128^3 ... 96^3) and compared element by
  element with the oracle (relative L-inf <= 1e-5 fp32 / 1e-12 fp64, ring bit-exact).  The grids
  are sized so the oracle does about 2e10 tap-updates per case; the three highest-order 3D box
  stencils (343-729 taps) use a thinner stream extent and T = 400/200/100 to stay in that budget
  (their b_T is 1: every sweep is the same one-step kernel, so a longer T adds no new code path).
* The headline workload (star2d1r fp32 16384^2, T = 1000) in bench.py's tuned configuration,
  compared on four 96 x 96 blocks of outputs (corner, edge, centre, and a block straddling a tile
  seam and a stream-block seam) -- 36,864 cells, each the oracle's exact full-grid value: the oracle
  runs on the dependency cone of each block (the block +- (T+1) rad, clipped to the array; a
  clipped side is the true ring).
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.float64: 1e-12}
NP = {torch.float32: np.float32, torch.float64: np.float64}

# interior size of the reduced grid (2D: n x n, 3D: (z, y, x)) and T
CASES = {
    "star2d1r": (2048, 1000), "j2d5pt": (2048, 1000), "star2d2r": (1536, 1000), "j2d9pt": (1536, 1000),
    "star2d3r": (1280, 1000), "star2d4r": (1152, 1000), "box2d1r": (1536, 1000), "box2d2r": (1024, 1000),
    "box2d3r": (768, 1000), "box2d4r": (640, 1000),
    "star3d1r": ((128, 128, 128), 1000), "star3d2r": ((112, 112, 112), 1000), "star3d3r": ((96, 96, 96), 1000),
    "star3d4r": ((96, 96, 96), 1000), "box3d1r": ((96, 96, 96), 1000), "j3d27pt": ((96, 96, 96), 1000),
    "box3d2r": ((48, 96, 128), 400), "box3d3r": ((32, 80, 128), 200), "box3d4r": ((24, 80, 128), 100),
}


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
    n, T = CASES[name]
    interior = (n, n) if ndim == 2 else n
    ext = tuple(v + 2 * rad for v in interior)
    full = (16384 + 2 * rad,) * 2 if ndim == 2 else (512 + 2 * rad,) * 3
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    pick = st.plan_config(full, 1000)                       # the planner's (b_T, vec) at BASELINE size
    cfg = st.plan_config(ext, T, {"bT": pick["bT"], "vec": pick["vec"]})   # h for this grid
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


def test_full_size_headline_blocks(an5d):
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
    st.run(a, b, T, cfg)
    torch.cuda.synchronize()
    out = b.cpu().numpy()
    geo = st.describe(ext, cfg)
    K = 96
    seam_x = rad + geo["compute"][0] * 7 - K // 2           # straddles the tile 6 | tile 7 seam
    seam_y = rad + cfg["h"] * 9 - K // 2                     # straddles stream blocks 8 | 9
    M = (T + 1) * rad
    for (y0b, x0b) in [(rad, rad), (rad, n // 2), (n // 2, n // 2), (seam_y, seam_x)]:
        y1b, x1b = y0b + K, x0b + K
        wy0, wy1 = max(0, y0b - M), min(ext[0], y1b + M)
        wx0, wx1 = max(0, x0b - M), min(ext[1], x1b + M)
        win = np.ascontiguousarray(g[wy0:wy1, wx0:wx1])
        exp = oracle.run(win, rad, shape, tab, div, T, np.float32)[y0b - wy0:y1b - wy0, x0b - wx0:x1b - wx0]
        got = out[y0b:y1b, x0b:x1b]
        err = np.abs(got.astype(np.float64) - exp).max() / np.abs(exp).max()
        assert err <= 1e-5, ((y0b, x0b), err, cfg)
