"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Acceptance (BASELINE.json north_star): relative L-inf (normwise, over the interior, SURVEY C-11)
<= 1e-5 for fp32 and <= 1e-12 for fp64; the ring compared bit-exactly; blocking bookkeeping
bit-exact -- checked by (i) exact-integer mode (+-1 taps, inputs in {-1,0,1}, T capped so every
partial sum is an exactly representable integer: any order of summation gives the same bits, so
GPU == oracle bit-for-bit and any halo/index/mask bug shows) and (ii) per-sweep write-count maps
(every interior cell stored exactly once, ring never).
"""
import os

import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.float64: 1e-12}
NP = {torch.float32: np.float32, torch.float64: np.float64}


def rel_linf(got, exp, rad):
    core = tuple(slice(rad, e - rad) for e in exp.shape)
    den = np.abs(exp[core]).max()
    return np.abs(got[core].astype(np.float64) - exp[core].astype(np.float64)).max() / max(den, 1e-300)


def ring_equal(got, exp, rad):
    mask = np.ones(exp.shape, bool)
    mask[tuple(slice(rad, e - rad) for e in exp.shape)] = False
    return np.array_equal(got[mask], exp[mask])


def gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg=None):
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_grid(g.shape, rad, dtype)
    b.fill_(float("nan"))
    st.run(a, b, T, cfg)
    torch.cuda.synchronize()
    return b.cpu().numpy(), st


def small_ext(ndim, rad):
    # spans several tiles in every blocked dim + ragged tails: 2D >= 5 vec-8 tiles across (256-cell
    # tiles), so interior (non-EDGE) units run too; 3D: >= 4 tiles across in y and x (64 x 32 and
    # 128 x 32 tiles)
    return (61 + 2 * rad, 1301 + 2 * rad) if ndim == 2 else (23 + 2 * rad, 131 + 2 * rad, 509 + 2 * rad)


def configs_for(an5d, st, ext, ndim, direct=0):
    """A spread of available (bT, vec, layout) configurations for this stencil, with short stream
    blocks so several stream blocks (and interior + edge units) are exercised.  2D: one warp per
    tile and the two-warp level split (n_thr = 64); 3D: the default 256-thread layout and the
    512-thread layouts (n_thr = 512: 64-wide fp64 / 128-wide fp32 tiles) where they are built."""
    out = []
    for n_thr in ((32, 64) if ndim == 2 and not direct else (0,) if ndim == 2 else (256, 512)):
        for vec in (1, 2, 4, 8):
            bts = []
            for bT in range(1, 11):
                try:
                    st.describe(ext, {"bT": bT, "vec": vec, "h": 16, "direct": direct, "n_thr": n_thr})
                    bts.append(bT)
                except an5d.AN5DError:
                    pass
            if bts:
                picks = sorted({bts[0], bts[len(bts) // 2], bts[-1]})
                out += [{"bT": b, "vec": vec, "h": 16 if ndim == 2 else 8, "direct": direct, "n_thr": n_thr}
                        for b in picks]
    return out


BENCH = sorted(inputs.BENCHMARKS)


@pytest.mark.parametrize("name", BENCH)
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_random_parity_all_configs(an5d, name, dtype):
    """Uniform [0,1) inputs, dyadic (or j-stencil integer/divisor) coefficients; every instance
    family; T in {1, bT, bT+1, 2bT+3}."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    cfgs = configs_for(an5d, st, ext, ndim)
    assert cfgs, f"no kernel instance for {name}"
    for cfg in cfgs:
        bT = cfg["bT"]
        for T in sorted({1, bT, bT + 1, 2 * bT + 3}):
            got, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
            exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
            assert ring_equal(got, exp, rad), (cfg, T)
            err = rel_linf(got, exp, rad)
            assert err <= TOL[dtype], (name, cfg, T, err)


def _exact_T(ndim, rad, shape, T_want, dtype):
    taps = (2 * rad + 1) ** ndim if shape == inputs.BOX else 2 * ndim * rad + 1
    lim = 2.0 ** (24 if dtype == torch.float32 else 53)
    T = 0
    bound = 1.0
    while T < T_want and bound * taps < lim:
        bound *= taps
        T += 1
    return T


@pytest.mark.parametrize("name", BENCH)
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_exact_integer_bit_identical(an5d, name, dtype):
    """+-1 taps, inputs in {-1,0,1}: every partial sum is an exact integer (< 2^24 / 2^53), so the
    GPU result must equal the oracle bit-for-bit whatever the summation order -- pins tile/halo
    indices, boundary masks and the sweep schedule exactly."""
    ndim, rad, shape, _, _ = inputs.benchmark_problem(name)
    if shape == inputs.GRAD:
        pytest.skip("gradient2d is not linear; its bit-exact check is test_gradient2d_bit_identical")
    tab, div = inputs.coeff_table(ndim, rad, shape, seed=99, kind="pm1")
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(1234, ext, kind="pm")
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    for cfg in configs_for(an5d, st, ext, ndim):
        T = _exact_T(ndim, rad, shape, 2 * cfg["bT"] + 3, dtype)
        if T < 1:
            continue
        got, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
        exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
        assert np.array_equal(got, exp), (name, cfg, T)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_gradient2d_bit_identical(an5d, dtype):
    """gradient2d (Table 2, NEXT N3) on the direct-gather kernel: every operation is
    individually rounded in the oracle's order (IEEE sqrt and division), so the GPU result equals
    the oracle BIT FOR BIT at every (b_T, vec), on ragged grids spanning several tiles, for
    T in {1, b_T, b_T + 1, 2 b_T + 3, 40} -- and every interior cell is stored once per sweep."""
    ndim, rad, shape, tab, c0 = inputs.benchmark_problem("gradient2d")
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED + 7, ext)
    st = an5d.Stencil(ndim, rad, shape, tab, c0, dtype)
    cfgs = configs_for(an5d, st, ext, ndim, direct=1)
    assert cfgs, "no gradient2d instance"
    for cfg in cfgs:
        bT = cfg["bT"]
        for T in sorted({1, bT, bT + 1, 2 * bT + 3, 40}):
            got, _ = gpu_run(an5d, ndim, rad, shape, tab, c0, g, T, dtype, cfg)
            exp = oracle.run(g, rad, shape, tab, c0, T, NP[dtype])
            assert np.array_equal(got, exp), (cfg, T, rel_linf(got, exp, rad))
        a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
        b = an5d.empty_grid(ext, rad, dtype)
        wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
        st.copy_ring(a, b)
        st.sweep(a, b, bT, cfg, write_count=wc)
        torch.cuda.synchronize()
        w = wc.cpu().numpy()
        core = tuple(slice(rad, e - rad) for e in ext)
        assert np.all(w[core] == 1), cfg
        w[core] = 0
        assert not w.any(), cfg


@pytest.mark.parametrize("name,dtype", [("star2d2r", torch.float32), ("star3d1r", torch.float64)])
def test_set_comm_single_rank(an5d, name, dtype):
    """an5d_set_comm: the library creates its own NCCL communicator; with one
    rank the slab is the whole array and the run is bit-identical to a plain run; detaching
    restores plain runs."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    ref, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, 11, dtype, {"bT": 2})
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    st.set_comm(an5d.comm_unique_id(), 0, 1, ext[0], 0, 0)
    a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_grid(ext, rad, dtype)
    st.run(a, b, 11, {"bT": 2})
    torch.cuda.synchronize()
    assert np.array_equal(b.cpu().numpy(), ref)
    st.set_comm(None)
    a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
    st.run(a, b, 11, {"bT": 2})
    torch.cuda.synchronize()
    assert np.array_equal(b.cpu().numpy(), ref)


OS_CASES = [(n, d) for n in ("star3d2r", "star3d3r", "star3d4r", "box3d2r", "box3d3r", "box3d4r")
            for d in (torch.float32, torch.float64)] + [(n, d) for n in ("box3d1r", "j3d27pt")
                                                        for d in (torch.float32, torch.float64)]


@pytest.mark.parametrize("name,dtype", OS_CASES)
def test_output_stationary_bt1(an5d, name, dtype):
    """Output-stationary b_T = 1 tiles (kernel3d.cuh OS): threads cover only the 64 x 32 compute
    region, x/y neighbours come from the staged plane.  Same per-cell arithmetic as the default
    layout, so BIT-IDENTICAL to it; within tolerance of the oracle; exact-integer bit-identical;
    every interior cell stored once (ragged grids, several tiles each way)."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    A = 4 if dtype == torch.float32 else 2
    hxo = -(-rad // A) * A
    cfg = {"bT": 1, "vec": 2, "h": 8, "n_thr": 256, "bS": [32 + 2 * rad, 64 + 2 * rad]}
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    d = st.describe(ext, cfg)
    assert d["bS_loaded"] == [32 + 2 * rad, 64 + 2 * hxo] and d["compute"] == [32, 64], d
    for T in (1, 2, 5):
        got, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
        ref, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, {"bT": 1, "vec": 2, "h": 8, "n_thr": 256,
                                                                          "bS": [32, 0]})
        assert np.array_equal(got, ref), (name, T)
        exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
        assert ring_equal(got, exp, rad) and rel_linf(got, exp, rad) <= TOL[dtype], (name, T)
    tabx, divx = inputs.coeff_table(ndim, rad, shape, seed=99, kind="pm1")
    gx = inputs.global_grid(1234, ext, kind="pm")
    T = _exact_T(ndim, rad, shape, 3, dtype)
    got, _ = gpu_run(an5d, ndim, rad, shape, tabx, divx, gx, T, dtype, cfg)
    assert np.array_equal(got, oracle.run(gx, rad, shape, tabx, divx, T, NP[dtype])), (name, T)
    a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_grid(ext, rad, dtype)
    wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
    st.copy_ring(a, b)
    st.sweep(a, b, 1, cfg, write_count=wc)
    torch.cuda.synchronize()
    w = wc.cpu().numpy()
    core = tuple(slice(rad, e - rad) for e in ext)
    assert np.all(w[core] == 1)
    w[core] = 0
    assert not w.any()


OY_CASES = [("star3d1r", torch.float32, 4, 256, False), ("star3d2r", torch.float32, 2, 256, False),
            ("box3d1r", torch.float32, 2, 256, False), ("star3d1r", torch.float64, 3, 512, False),
            ("star3d2r", torch.float64, 2, 512, False), ("box3d1r", torch.float64, 2, 512, False),
            ("star3d1r", torch.float64, 3, 512, True), ("star3d2r", torch.float64, 2, 512, True),
            ("box3d1r", torch.float64, 2, 512, True)]


@pytest.mark.parametrize("name,dtype,bmax,n_thr,xstage", OY_CASES)
def test_y_staged_tiles(an5d, name, dtype, bmax, n_thr, xstage):
    """y-staged tiles (kernel3d.cuh OS bit 0): the TMA box adds rad rows above and below, so the
    threads' y halo shrinks to (b_T - 1) rad; with x staging (bit 1, fp64 512-thread layout) level 1
    also reads its x neighbours from the stage.  Bit-identical to the default layout at every b_T,
    within tolerance of the oracle, exact-integer bit-identical, write counts once per sweep."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    tabx, divx = inputs.coeff_table(ndim, rad, shape, seed=99, kind="pm1")
    gx = inputs.global_grid(1234, ext, kind="pm")
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    A = 4 if dtype == torch.float32 else 2
    rup = lambda v: -(-v // A) * A
    for bT in range(1, bmax + 1):
        # x staging: loaded width 64 + 2 rup(rad), compute width 64 - 2 rup((b_T - 1) rad); the
        # logical b_S = compute + 2 b_T rad names the layout (an5d.h an5d_config)
        bsx = (64 - 2 * rup((bT - 1) * rad) + 2 * bT * rad) if xstage else 0
        if xstage and bsx == 64 - 2 * rup(bT * rad) + 2 * bT * rad:
            continue   # same compute region as the unstaged layout at this b_T: nothing to test
        cfg = {"bT": bT, "vec": 2, "h": 8, "n_thr": n_thr, "bS": [32 + 2 * rad, bsx]}
        d = st.describe(ext, cfg)
        assert d["bS_loaded"][0] == 32 + 2 * rad and d["compute"][0] == 32 - 2 * (bT - 1) * rad, d
        if xstage:
            assert d["bS_loaded"][1] == 64 + 2 * rup(rad) and d["compute"][1] == 64 - 2 * rup((bT - 1) * rad), d
        for T in sorted({1, bT, 2 * bT + 3}):
            got, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
            ref, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, dict(cfg, bS=[32, 0]))
            assert np.array_equal(got, ref), (name, bT, T, xstage)
            exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
            assert ring_equal(got, exp, rad) and rel_linf(got, exp, rad) <= TOL[dtype], (name, bT, T)
        T = _exact_T(ndim, rad, shape, 2 * bT + 3, dtype)
        got, _ = gpu_run(an5d, ndim, rad, shape, tabx, divx, gx, T, dtype, cfg)
        assert np.array_equal(got, oracle.run(gx, rad, shape, tabx, divx, T, NP[dtype])), (name, bT, T)
        a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
        b = an5d.empty_grid(ext, rad, dtype)
        wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
        st.copy_ring(a, b)
        st.sweep(a, b, bT, cfg, write_count=wc)
        torch.cuda.synchronize()
        w = wc.cpu().numpy()
        core = tuple(slice(rad, e - rad) for e in ext)
        assert np.all(w[core] == 1), bT
        w[core] = 0
        assert not w.any(), bT


# x-pair 3D tiles (kernel3d.cuh Kernel3DTraits::XPAIR): fp32 layouts without x staging whose
# b_T rad = 2 mod 4 load an x halo of exactly b_T rad (the TMA box starts on the 16-byte boundary
# 2 cells before the window and is 4 cells wider) and store 8-byte cell pairs; (stencil, b_T,
# loaded tile height bS_y naming the layout: 32 default, 32 + 2 rad y-staged, 64 cluster pair)
XPAIR_CASES = [("star3d1r", 2, 32), ("star3d1r", 2, 34), ("star3d1r", 2, 64), ("box3d1r", 2, 32),
               ("box3d1r", 2, 34), ("j3d27pt", 2, 64), ("star3d2r", 1, 32), ("box3d2r", 1, 32)]


@pytest.mark.parametrize("name,bT,bsy", XPAIR_CASES)
def test_xpair_tiles(an5d, name, bT, bsy):
    """Geometry (bit-exact): loaded x halo b_T rad, compute width 64 - 2 b_T rad, tile count
    ceil(I_x / C_x); exact-integer GPU == oracle bit for bit; random inputs within
    tolerance; every interior cell stored exactly once per sweep (ragged grid, several x tiles,
    compute regions 2 cells off a 16-byte boundary)."""
    dtype = torch.float32
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    cfg = {"bT": bT, "vec": 2, "h": 8, "n_thr": 256, "bS": [bsy, 0]}
    d = st.describe(ext, cfg)
    assert (bT * rad) % 4 == 2
    assert d["halo_loaded"][1] == bT * rad and d["compute"][1] == 64 - 2 * bT * rad, d
    assert d["n_tiles"][1] == -(-(ext[2] - 2 * rad) // (64 - 2 * bT * rad)), d
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    for T in sorted({bT, 2 * bT + 1}):
        got, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
        exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
        assert ring_equal(got, exp, rad) and rel_linf(got, exp, rad) <= TOL[dtype], (name, bT, bsy, T)
    tabx, divx = inputs.coeff_table(ndim, rad, shape, seed=99, kind="pm1")
    gx = inputs.global_grid(1234, ext, kind="pm")
    T = _exact_T(ndim, rad, shape, 2 * bT + 3, dtype)
    got, _ = gpu_run(an5d, ndim, rad, shape, tabx, divx, gx, T, dtype, cfg)
    assert np.array_equal(got, oracle.run(gx, rad, shape, tabx, divx, T, NP[dtype])), (name, bT, bsy, T)
    a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_grid(ext, rad, dtype)
    wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
    st.copy_ring(a, b)
    st.sweep(a, b, bT, cfg, write_count=wc)
    torch.cuda.synchronize()
    w = wc.cpu().numpy()
    core = tuple(slice(rad, e - rad) for e in ext)
    assert np.all(w[core] == 1), (name, bT, bsy)
    w[core] = 0
    assert not w.any(), (name, bT, bsy)


CLUSTER_CASES = [("star3d1r", torch.float32, 4, 256, (2, 4)), ("star3d2r", torch.float32, 2, 256, (2,)),
                 ("box3d1r", torch.float32, 2, 256, (2,)), ("j3d27pt", torch.float32, 2, 256, (2,)),
                 ("star3d1r", torch.float64, 3, 256, (2,)), ("star3d1r", torch.float64, 3, 512, (2,)),
                 ("star3d2r", torch.float64, 2, 512, (2,)), ("box3d1r", torch.float64, 2, 512, (2,))]


@pytest.mark.parametrize("name,dtype,bmax,n_thr,cls", CLUSTER_CASES)
def test_cluster_halo_sharing(an5d, name, dtype, bmax, n_thr, cls):
    """3D thread-block clusters (NEXT N2): CL blocks stacked along y share their y halos through
    DSMEM -- one tile of CL x 32 rows.  Per cell the arithmetic is unchanged, so every run is
    BIT-IDENTICAL to the one-block layout (32-row tiles) with the same b_T, matches the oracle
    within tolerance on random inputs and bit-for-bit in exact-integer mode, and stores every
    interior cell once per sweep (ragged grids: several cluster tiles in y, partial last one)."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    tabx, divx = inputs.coeff_table(ndim, rad, shape, seed=99, kind="pm1")
    gx = inputs.global_grid(1234, ext, kind="pm")
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    for cl in cls:
        for bT in range(1, bmax + 1):
            cfg = {"bT": bT, "vec": 2, "h": 8, "n_thr": n_thr, "bS": [32 * cl, 0]}
            d = st.describe(ext, cfg)
            assert d["bS_loaded"][0] == 32 * cl and d["grid_blocks"] % cl == 0, d
            ref_cfg = dict(cfg, bS=[32, 0])
            for T in sorted({1, bT, 2 * bT + 3}):
                got, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
                ref, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, ref_cfg)
                assert np.array_equal(got, ref), (name, cl, bT, T)
                exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
                assert ring_equal(got, exp, rad) and rel_linf(got, exp, rad) <= TOL[dtype], (name, cl, bT, T)
            T = _exact_T(ndim, rad, shape, 2 * bT + 3, dtype)
            got, _ = gpu_run(an5d, ndim, rad, shape, tabx, divx, gx, T, dtype, cfg)
            assert np.array_equal(got, oracle.run(gx, rad, shape, tabx, divx, T, NP[dtype])), (name, cl, bT, T)
            a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
            b = an5d.empty_grid(ext, rad, dtype)
            wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
            st.copy_ring(a, b)
            st.sweep(a, b, bT, cfg, write_count=wc)
            torch.cuda.synchronize()
            w = wc.cpu().numpy()
            core = tuple(slice(rad, e - rad) for e in ext)
            assert np.all(w[core] == 1), (cl, bT)
            w[core] = 0
            assert not w.any(), (cl, bT)


# the default build has direct-gather instances for BASELINE config 4 only (box2d2r fp32); the
# full build (AN5D_FULL_BUILD=1) adds box2d1r-4r fp32/fp64, which this test then also covers
@pytest.mark.parametrize("name,dtype", [("box2d2r", torch.float32)] + [
    (n, d) for n in ("box2d1r", "box2d2r", "box2d3r", "box2d4r") for d in (torch.float32, torch.float64)
    if os.environ.get("AN5D_FULL_BUILD", "") not in ("", "0") and (n, d) != ("box2d2r", torch.float32)])
def test_direct_gather_variant(an5d, name, dtype):
    """Partial sums OFF (Table 1 "Otherwise"; BASELINE config 4): the direct-gather
    kernels match the oracle within tolerance on random inputs, bit-for-bit in exact-integer mode,
    and store every interior cell exactly once."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    cfgs = configs_for(an5d, st, ext, ndim, direct=1)
    assert cfgs, f"no direct instance for {name}"
    tabx, divx = inputs.coeff_table(ndim, rad, shape, seed=99, kind="pm1")
    gx = inputs.global_grid(1234, ext, kind="pm")
    for cfg in cfgs:
        bT = cfg["bT"]
        for T in sorted({1, bT, 2 * bT + 3}):
            got, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
            exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
            assert ring_equal(got, exp, rad), (cfg, T)
            assert rel_linf(got, exp, rad) <= TOL[dtype], (name, cfg, T)
        T = _exact_T(ndim, rad, shape, 2 * bT + 3, dtype)
        if T >= 1:
            got, _ = gpu_run(an5d, ndim, rad, shape, tabx, divx, gx, T, dtype, cfg)
            assert np.array_equal(got, oracle.run(gx, rad, shape, tabx, divx, T, NP[dtype])), (name, cfg, T)
        a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
        b = an5d.empty_grid(ext, rad, dtype)
        wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
        st.copy_ring(a, b)
        st.sweep(a, b, bT, cfg, write_count=wc)
        torch.cuda.synchronize()
        w = wc.cpu().numpy()
        core = tuple(slice(rad, e - rad) for e in ext)
        assert np.all(w[core] == 1), cfg
        w[core] = 0
        assert not w.any(), cfg


@pytest.mark.parametrize("name", ["star2d1r", "box2d3r", "j2d9pt", "star3d2r", "box3d1r", "box3d4r"])
def test_write_count_map(an5d, name):
    """One sweep: every interior cell stored exactly once, ring cells never (S:213 coverage and
    disjointness of compute regions)."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    g = inputs.global_grid(5, ext)
    a = an5d.to_grid(torch.from_numpy(g.astype(np.float32)).cuda(), rad)
    b = an5d.empty_grid(ext, rad, torch.float32)
    for cfg in configs_for(an5d, st, ext, ndim):
        wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
        st.copy_ring(a, b)
        st.sweep(a, b, cfg["bT"], cfg, write_count=wc)
        torch.cuda.synchronize()
        w = wc.cpu().numpy()
        core = tuple(slice(rad, e - rad) for e in ext)
        assert np.all(w[core] == 1), cfg
        w[core] = 0
        assert not w.any(), cfg


def test_baseline_config1_full(an5d):
    """BASELINE config 1: star2d1r fp32 512^2, T=100, bT=4 -- full grid against the oracle."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem("star2d1r")
    ext = (512 + 2, 512 + 2)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    got, st = gpu_run(an5d, ndim, rad, shape, tab, div, g, 100, torch.float32, {"bT": 4})
    exp = oracle.run(g, rad, shape, tab, div, 100, np.float32)
    assert ring_equal(got, exp, rad)
    assert rel_linf(got, exp, rad) <= 1e-5


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_edge_cases(an5d, dtype):
    """Degenerate sizes: a single interior cell, interior smaller than one tile, one interior plane,
    T = 0, T < bT."""
    for ndim, rad, shape in [(2, 1, inputs.STAR), (2, 3, inputs.BOX), (3, 1, inputs.BOX), (3, 2, inputs.STAR)]:
        tab, div = inputs.coeff_table(ndim, rad, shape, seed=4)
        for n in ([1, 1], [3, 5], [1, 40]) if ndim == 2 else ([1, 1, 1], [2, 3, 5], [9, 1, 70]):
            ext = tuple(v + 2 * rad for v in n)
            g = inputs.global_grid(8, ext)
            for T in (0, 1, 2, 5):
                got, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype)
                exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
                assert ring_equal(got, exp, rad)
                assert rel_linf(got, exp, rad) <= TOL[dtype], (ndim, rad, n, T)


def test_errors_before_launch(an5d):
    """Misaligned pitch / base -> AN5D_ERR_UNSUPPORTED with nothing written."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem("star2d1r")
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    a = torch.zeros(10, 13, device="cuda")          # pitch 13 floats: not 16-byte multiple
    b = torch.full((10, 13), 7.0, device="cuda")
    with pytest.raises(an5d.AN5DError) as e:
        st.run(a, b, 3)
    assert e.value.status == 5
    assert torch.all(b == 7.0)


def test_run_split_equals_single_run(an5d):
    """Checkpoint/resume semantics: run(T1) then run(T2) == run(T1+T2) bit-exactly when the sweep
    degrees coincide (both schedules are all-bT sweeps here)."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem("box2d1r")
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(3, ext)
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    cfg = {"bT": 3, "vec": 8, "h": 32}
    a = an5d.to_grid(torch.from_numpy(g.astype(np.float32)).cuda(), rad)
    b = an5d.empty_grid(ext, rad, torch.float32)
    st.run(a, b, 9, cfg)                      # 3 sweeps of 3 -> result in b
    full = b.clone()
    a2 = an5d.to_grid(torch.from_numpy(g.astype(np.float32)).cuda(), rad)
    b2 = an5d.empty_grid(ext, rad, torch.float32)
    st.run(a2, b2, 3, cfg)
    a3 = an5d.to_grid(b2, rad)
    b3 = an5d.empty_grid(ext, rad, torch.float32)
    st.run(a3, b3, 6, cfg)                    # schedule [3, 3] is even -> split: [3, 2, 1]
    torch.cuda.synchronize()
    err = rel_linf(b3.cpu().numpy(), full.cpu().numpy(), rad)
    assert err <= 1e-6


@pytest.mark.parametrize("name,n_int,T,bT,nslab", [
    ("star2d1r", (97, 131), 9, 4, 3),
    ("box2d2r", (61, 77), 7, 2, 2),
    ("star3d1r", (41, 37, 70), 7, 3, 3),
    ("j3d27pt", (33, 19, 45), 5, 2, 2),
])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_slab_loopback_bit_identical(an5d, name, n_int, T, bT, nslab, dtype):
    """Multi-GPU slab bookkeeping on one device (SURVEY §4 loopback mode): the streaming dim split
    into slabs with ghost planes, an5d_sweep in slab mode, ghosts exchanged by device copies.  The
    gathered owned planes must equal the single-domain an5d_run bit-for-bit (same per-cell
    arithmetic) and the oracle within tolerance."""
    from paper_2001_01473_b200 import slab
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    gext = tuple(v + 2 * rad for v in n_int)
    g = inputs.global_grid(inputs.DEFAULT_SEED, gext)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    cfg = st.plan_config(gext, T, {"bT": bT, "h": 8})
    ref, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
    parts = slab.partition(gext[0], rad, nslab, cfg["bT"] * rad)
    bufs = []
    for s in parts:
        loc = g[s.loc_lo:s.loc_hi]
        a = an5d.to_grid(torch.from_numpy(loc.astype(NP[dtype])).cuda(), rad)
        b = an5d.empty_grid(loc.shape, rad, dtype)
        b.fill_(float("nan"))
        bufs.append((a, b))
    outs = slab.run_loopback(st, parts, bufs, T, cfg)
    torch.cuda.synchronize()
    got = np.concatenate([o.cpu().numpy()[s.out_lo:s.out_hi] for s, o in zip(parts, outs)])
    assert np.array_equal(got, ref[rad:gext[0] - rad])
    exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
    full = ref.copy()
    full[rad:gext[0] - rad] = got
    assert rel_linf(full, exp, rad) <= TOL[dtype]


@pytest.mark.parametrize("name,dtype", [("star2d1r", torch.float32), ("box2d2r", torch.float64),
                                        ("star3d1r", torch.float32)])
def test_tune_then_run(an5d, name, dtype):
    """an5d_tune (model top-k + measured pick) returns a feasible configuration that
    honours the hint, leaves grid_in untouched, and the run with it matches the oracle."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_grid(ext, rad, dtype)
    a0 = a.clone()
    cfg = st.tune(a, b, 7, {"h": 16}, top_k=3)
    torch.cuda.synchronize()
    assert cfg["h"] == 16 and cfg["bT"] >= 1 and cfg["seconds_per_cell_step"] > 0
    assert torch.equal(a, a0)
    cfg.pop("seconds_per_cell_step")
    st.run(a, b, 7, cfg)
    torch.cuda.synchronize()
    exp = oracle.run(g, rad, shape, tab, div, 7, NP[dtype])
    got = b.cpu().numpy()
    assert ring_equal(got, exp, rad)
    assert rel_linf(got, exp, rad) <= TOL[dtype]


@pytest.mark.parametrize("name,dtype,cfg", [
    ("star2d1r", torch.float32, {"bT": 3, "h": 8, "vec": 8}),
    ("star2d1r", torch.float32, {"bT": 7, "h": 16, "vec": 8}),
    ("box2d2r", torch.float64, {"bT": 2, "h": 8, "vec": 4}),
    ("j2d5pt", torch.float32, {"bT": 4, "h": 8, "vec": 8}),
    ("star2d1r", torch.float32, {"bT": 7, "h": 16, "vec": 8, "n_thr": 64}),
    ("star2d1r", torch.float32, {"bT": 3, "h": 8, "vec": 8, "n_thr": 64}),
    ("star2d1r", torch.float32, {"bT": 4, "h": 8, "vec": 8, "n_thr": 64}),
])
def test_stream_block_runs(an5d, name, dtype, cfg, monkeypatch):
    """2D run schedule (an5d_host.cu build_runs_2d: x-edge singles, y-edge singles, one round of
    long runs of consecutive stream blocks per interior tile, a tail of singles).  The run table is
    shaped for 4 warps (AN5D_RUN_WARPS) so an oracle-sized grid gets runs of ~10-20 stream blocks:
    result within tolerance of the oracle, bit-identical to the plain one-stream-block-per-unit
    schedule (AN5D_RUN_FRAC=0: same per-row arithmetic), every interior cell stored exactly once."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = (203 + 2 * rad, 1100 + 2 * rad)   # >= 4 tiles across (interior tiles exist), ~25 stream blocks
    g = inputs.global_grid(77, ext)
    T = 2 * cfg["bT"] + 1
    monkeypatch.setenv("AN5D_RUN_WARPS", "4")
    got, st = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
    exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
    assert ring_equal(got, exp, rad)
    assert rel_linf(got, exp, rad) <= TOL[dtype], (name, cfg)
    monkeypatch.setenv("AN5D_RUN_FRAC", "0")
    plain, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
    assert np.array_equal(got, plain), (name, cfg)
    monkeypatch.delenv("AN5D_RUN_FRAC")
    # exact-integer mode: bit-identical to the oracle
    tabx, divx = inputs.coeff_table(ndim, rad, shape, seed=99, kind="pm1")
    gx = inputs.global_grid(1234, ext, kind="pm")
    Tx = _exact_T(ndim, rad, shape, T, dtype)
    gotx, _ = gpu_run(an5d, ndim, rad, shape, tabx, divx, gx, Tx, dtype, cfg)
    assert np.array_equal(gotx, oracle.run(gx, rad, shape, tabx, divx, Tx, NP[dtype])), (name, cfg, Tx)
    # one sweep with store counts (routes every unit through the EDGE loop, runs included)
    a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_grid(ext, rad, dtype)
    wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
    st.copy_ring(a, b)
    st.sweep(a, b, cfg["bT"], st.plan_config(ext, T, cfg), write_count=wc)
    torch.cuda.synchronize()
    w = wc.cpu().numpy()
    core = tuple(slice(rad, e - rad) for e in ext)
    assert np.all(w[core] == 1), cfg
    w[core] = 0
    assert not w.any(), cfg


@pytest.mark.parametrize("name,dtype,cfg", [
    ("star3d1r", torch.float32, {"bT": 3, "h": 4, "vec": 2}),
    ("box3d1r", torch.float64, {"bT": 2, "h": 4, "vec": 2}),
    ("star3d2r", torch.float32, {"bT": 2, "h": 4, "vec": 2}),
    ("star3d1r", torch.float64, {"bT": 3, "h": 4, "vec": 2, "n_thr": 512}),
    ("star3d2r", torch.float64, {"bT": 2, "h": 4, "vec": 2, "n_thr": 512}),
])
def test_stream_block_runs_3d(an5d, name, dtype, cfg, monkeypatch):
    """3D run schedule (build_runs_3d): long runs forced by shaping the table for 2 blocks; oracle
    parity, bit-identical to the plain schedule, exact-integer mode, store counts once."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = (41 + 2 * rad, 150 + 2 * rad, 530 + 2 * rad)   # >= 4 tiles in y and x (interior tiles), ~10 stream blocks
    g = inputs.global_grid(78, ext)
    T = 2 * cfg["bT"] + 1
    monkeypatch.setenv("AN5D_RUN_WARPS", "2")
    got, st = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
    exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
    assert ring_equal(got, exp, rad)
    assert rel_linf(got, exp, rad) <= TOL[dtype], (name, cfg)
    monkeypatch.setenv("AN5D_RUN_FRAC", "0")
    plain, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
    assert np.array_equal(got, plain), (name, cfg)
    monkeypatch.delenv("AN5D_RUN_FRAC")
    tabx, divx = inputs.coeff_table(ndim, rad, shape, seed=99, kind="pm1")
    gx = inputs.global_grid(1234, ext, kind="pm")
    Tx = _exact_T(ndim, rad, shape, T, dtype)
    gotx, _ = gpu_run(an5d, ndim, rad, shape, tabx, divx, gx, Tx, dtype, cfg)
    assert np.array_equal(gotx, oracle.run(gx, rad, shape, tabx, divx, Tx, NP[dtype])), (name, cfg, Tx)
    a = an5d.to_grid(torch.from_numpy(g.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_grid(ext, rad, dtype)
    wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
    st.copy_ring(a, b)
    st.sweep(a, b, cfg["bT"], st.plan_config(ext, T, cfg), write_count=wc)
    torch.cuda.synchronize()
    w = wc.cpu().numpy()
    core = tuple(slice(rad, e - rad) for e in ext)
    assert np.all(w[core] == 1), cfg
    w[core] = 0
    assert not w.any(), cfg


def _bench_cfg(st, a, b, T):
    """The launch configuration bench.py times: the measured top-5 pick (an5d_tune)."""
    cfg = st.tune(a, b, T, None, top_k=5)
    cfg.pop("seconds_per_cell_step", None)
    return cfg


@pytest.mark.parametrize("name", ["star2d1r", "star2d4r", "box2d2r", "star3d2r", "box3d1r"])
def test_full_size_linear_field_exact(an5d, name):
    """Full BASELINE size and T = 1000 in bench.py's tuned configuration (fp64): a symmetric stencil
    with sum 1 maps a linear field to itself (oracle pin `test_linear_field_fixed_point`), and with
    dyadic coefficients and a dyadic field every product and partial sum is exact in fp64 -- so the
    result must equal the input bit-for-bit in EVERY cell.  A wrong tap offset, halo, tile seam,
    stream-block seam, ring mask or run boundary anywhere in the 16384^2 / 512^3 grid breaks it."""
    ndim, rad, shape, _, _ = inputs.benchmark_problem(name)
    tab, div = inputs.coeff_table(ndim, rad, shape, seed=5, symmetric=True)
    n = 16384 if ndim == 2 else 512
    ext = (n + 2 * rad,) * ndim
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float64)
    a = an5d.empty_grid(ext, rad, torch.float64)
    b = an5d.empty_grid(ext, rad, torch.float64)
    idx = [torch.arange(e, dtype=torch.float64, device="cuda") for e in ext]
    if ndim == 2:
        lin = 1.0 + (2 * idx[0][:, None] + idx[1][None, :]) * 2.0 ** -15
    else:
        lin = 1.0 + (3 * idx[0][:, None, None] + 2 * idx[1][None, :, None] + idx[2][None, None, :]) * 2.0 ** -12
    a.copy_(lin)
    cfg = _bench_cfg(st, a, b, 1000)
    a.copy_(lin)
    b.fill_(float("nan"))   # every cell of the result must be written by this run
    st.run(a, b, 1000, cfg)
    torch.cuda.synchronize()
    assert torch.equal(b, lin), (name, cfg, float((b - lin).abs().max()))


@pytest.mark.parametrize("name,dtype,bT,vec", [("star2d1r", torch.float32, 7, 8), ("star2d1r", torch.float32, 8, 8),
                                               ("star2d1r", torch.float32, 3, 8), ("star2d1r", torch.float32, 2, 8),
                                               ("j2d5pt", torch.float32, 5, 8), ("j2d5pt", torch.float32, 6, 8)])
def test_level_split_bit_identical(an5d, name, dtype, bT, vec):
    """The two-warp level split (n_thr = 64: warp 0 levels 1..b_T/2, warp 1 the rest, rows handed
    over through a shared-memory queue) does exactly the one-warp kernel's per-cell arithmetic, so
    its result is the same bits -- on a grid with interior and edge units, several stream blocks,
    a reduced-degree sweep (degree 1 runs the one-warp instance) -- and matches the oracle."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = (157 + 2 * rad, 1500 + 2 * rad)
    g = inputs.global_grid(91, ext)
    T = 2 * bT + 1
    one, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, {"bT": bT, "vec": vec, "h": 24, "n_thr": 32})
    two, st = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, {"bT": bT, "vec": vec, "h": 24, "n_thr": 64})
    assert st.plan_config(ext, T, {"bT": bT, "vec": vec, "h": 24, "n_thr": 64})["n_thr"] == 64
    assert np.array_equal(one, two), (name, bT)
    exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
    assert ring_equal(two, exp, rad)
    assert rel_linf(two, exp, rad) <= TOL[dtype]


@pytest.mark.parametrize("name,n_int,T,bT,nslab,dtype,extra", [
    ("star2d1r", (301, 1000), 9, 4, 3, torch.float32, {}),
    ("star2d1r", (301, 1000), 15, 7, 2, torch.float32, {"n_thr": 64}),
    ("box2d2r", (121, 700), 7, 2, 2, torch.float64, {}),
    ("star3d1r", (61, 70, 130), 7, 3, 3, torch.float32, {}),
    ("star3d2r", (49, 40, 150), 5, 2, 2, torch.float64, {"n_thr": 512}),
    ("j3d27pt", (41, 37, 70), 4, 1, 2, torch.float32, {}),
])
def test_fused_halo_loopback_bit_identical(an5d, name, n_int, T, bT, nslab, dtype, extra):
    """Fused halo exchange (NEXT N1) on one device: every slab on its own stream, the sweep
    kernels store the boundary planes straight into the neighbours' ghost planes (an5d_sweep_peer)
    and 32-bit stream flags order the slabs (an5d_stream_signal / an5d_stream_wait).  The
    gathered owned planes equal the single-domain an5d_run bit for bit (b_T 1 with an even sweep
    count and reduced-degree sweeps included) and the oracle within tolerance."""
    from paper_2001_01473_b200 import slab
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    gext = tuple(v + 2 * rad for v in n_int)
    g = inputs.global_grid(inputs.DEFAULT_SEED, gext)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    cfg = st.plan_config(gext, T, dict({"bT": bT, "h": 8}, **extra))
    ref, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
    parts = slab.partition(gext[0], rad, nslab, cfg["bT"] * rad)
    bufs = []
    for s in parts:
        loc = g[s.loc_lo:s.loc_hi]
        a = an5d.to_grid(torch.from_numpy(loc.astype(NP[dtype])).cuda(), rad)
        b = an5d.empty_grid(loc.shape, rad, dtype)
        b.fill_(float("nan"))
        bufs.append((a, b))
    outs = slab.loopback_fused(st, parts, bufs, T, cfg)
    got = np.concatenate([o.cpu().numpy()[s.out_lo:s.out_hi] for s, o in zip(parts, outs)])
    assert np.array_equal(got, ref[rad:gext[0] - rad]), (name, cfg)
    exp = oracle.run(g, rad, shape, tab, div, T, NP[dtype])
    full = ref.copy()
    full[rad:gext[0] - rad] = got
    assert rel_linf(full, exp, rad) <= TOL[dtype]


def _ipc_worker(rank, ws, port, name, n_int, T, bT, dtype_name, out_path):
    import torch.distributed as dist
    import paper_2001_01473_b200 as an5d
    from paper_2001_01473_b200 import slab
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    torch.cuda.set_device(0)
    dtype = getattr(torch, dtype_name)
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    gext = tuple(v + 2 * rad for v in n_int)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    cfg = st.plan_config(gext, T, {"bT": bT, "h": 8})
    parts = slab.partition(gext[0], rad, ws, cfg["bT"] * rad)
    s = parts[rank]
    loc = inputs.global_grid(inputs.DEFAULT_SEED, gext)[s.loc_lo:s.loc_hi]
    a = an5d.to_grid(torch.from_numpy(loc.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_grid(loc.shape, rad, dtype)
    flag = torch.zeros(32, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    fl, opened = slab.connect_fused(parts, rank, (a, b), flag)
    dist.barrier()
    out = slab.run_fused(st, s, (a, b), T, cfg, fl, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    dist.barrier()
    owned = out.cpu().numpy()[s.out_lo:s.out_hi]
    res = [None] * ws
    dist.all_gather_object(res, owned)
    if rank == 0:
        np.save(out_path, np.concatenate(res))
    dist.barrier()
    for base in opened:
        an5d.ipc_close(base)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n_int,T,bT", [("star2d2r", (203, 600), 9, 3), ("star3d1r", (50, 40, 130), 7, 2)])
def test_fused_halo_ipc_two_processes(an5d, tmp_path, name, n_int, T, bT):
    """The fused exchange across PROCESSES (the multi-GPU deployment: one process per GPU): two
    ranks on one device map each other's slab buffers and flags with CUDA IPC (an5d_ipc_export /
    an5d_ipc_open) and run run_fused; the gathered result equals the single-domain an5d_run."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = str(tmp_path / "res.npy")
    mp.start_processes(_ipc_worker, args=(2, port, name, n_int, T, bT, "float32", out), nprocs=2,
                       start_method="spawn", join=True)
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    gext = tuple(v + 2 * rad for v in n_int)
    g = inputs.global_grid(inputs.DEFAULT_SEED, gext)
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    ref, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, torch.float32, st.plan_config(gext, T, {"bT": bT, "h": 8}))
    assert np.array_equal(np.load(out), ref[rad:gext[0] - rad])


@pytest.mark.parametrize("name,dtype,bT", [("star2d1r", torch.float32, 4), ("box3d1r", torch.float32, 2),
                                           ("star3d1r", torch.float64, 3)])
def test_cuda_graph_capture_bit_identical(an5d, name, dtype, bT):
    """The whole T-step run (ring copy, every sweep with its programmatic-dependent launch, the
    reduced-degree sweeps of the schedule) captured in a CUDA graph after one eager warm-up run
    and replayed twice from a re-initialised input: bit-identical to the eager run each time."""
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = small_ext(ndim, rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    T = 2 * bT + 1
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    cfg = st.plan_config(ext, T, {"bT": bT, "vec": 8 if ndim == 2 and dtype == torch.float32 else (4 if ndim == 2 else 2),
                                  "h": 16 if ndim == 2 else 8})
    ref, _ = gpu_run(an5d, ndim, rad, shape, tab, div, g, T, dtype, cfg)
    init = torch.from_numpy(g.astype(NP[dtype])).cuda()
    a = an5d.to_grid(init, rad)
    b = an5d.empty_grid(ext, rad, dtype)
    st.run(a, b, T, cfg)            # eager warm-up: run tables, occupancy, attributes cached
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        st.run(a, b, T, cfg)
    for _ in range(2):
        a.copy_(init)
        b.fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(b.cpu().numpy(), ref), (name, cfg)
