"""GPU parity of multi-field systems (NEXT N4: multi-output temporal blocking of a
multi-statement stencil) through the C ABI (an5d_create_system) against the system oracle.

* random fields, dyadic row-stochastic blocks: every (b_T, vec) instance, ragged 2D grids over
  several tiles, T in {1, b_T, b_T + 1, 2 b_T + 3}: relative L-inf <= 1e-5 / 1e-12 per field,
  rings bit-exact;
* exact-integer mode (+-1 blocks, inputs in {-1, 0, 1}): bit-identical to the oracle;
* a decoupled system (zero off-diagonal blocks) is bit-identical to two single-field runs;
* one sweep stores every interior cell of every field once, rings never;
* full T = 1000 at the planner's configuration (2048^2), element by element.
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.float64: 1e-12}
NP = {torch.float32: np.float32, torch.float64: np.float64}
EXT = (61 + 2, 1301 + 2)   # >= 5 vec-8 tiles across (interior units run) + ragged tails


def rel_linf(got, exp, rad):
    core = (slice(None),) + tuple(slice(rad, e - rad) for e in exp.shape[1:])
    den = np.abs(exp[core]).max()
    return np.abs(got[core].astype(np.float64) - exp[core].astype(np.float64)).max() / max(den, 1e-300)


def rings_equal(got, exp, rad):
    mask = np.ones(exp.shape[1:], bool)
    mask[tuple(slice(rad, e - rad) for e in exp.shape[1:])] = False
    return all(np.array_equal(got[f][mask], exp[f][mask]) for f in range(exp.shape[0]))


def run_system(an5d, ndim, rad, shape, tab, fields, T, dtype, cfg=None):
    st = an5d.System(ndim, rad, shape, tab, dtype)
    a = an5d.to_fields(torch.from_numpy(fields.astype(NP[dtype])).cuda(), rad)
    b = an5d.empty_fields(fields.shape[0], fields.shape[1:], rad, dtype)
    b.fill_(float("nan"))
    st.run(a, b, T, cfg)
    torch.cuda.synchronize()
    return b.cpu().numpy(), st


def configs(an5d, st, ext):
    out = []
    for vec in (2, 4, 8):
        for bT in range(1, 11):
            try:
                st.describe(ext, {"bT": bT, "vec": vec, "h": 16})
                out.append({"bT": bT, "vec": vec, "h": 16})
            except an5d.AN5DError:
                pass
    return out


@pytest.mark.parametrize("name", sorted(inputs.SYSTEMS))
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_system_random_parity(an5d, name, dtype):
    ndim, rad, shape, nf, tab = inputs.system_problem(name)
    f = inputs.system_fields(inputs.DEFAULT_SEED, nf, EXT)
    st = an5d.System(ndim, rad, shape, tab, dtype)
    cfgs = configs(an5d, st, EXT)
    assert cfgs, name
    for cfg in cfgs:
        bT = cfg["bT"]
        for T in sorted({1, bT, bT + 1, 2 * bT + 3}):
            got, _ = run_system(an5d, ndim, rad, shape, tab, f, T, dtype, cfg)
            exp = oracle.run_system(f, rad, shape, tab, T, NP[dtype])
            assert rings_equal(got, exp, rad), (cfg, T)
            assert rel_linf(got, exp, rad) <= TOL[dtype], (name, cfg, T, rel_linf(got, exp, rad))


@pytest.mark.parametrize("name", sorted(inputs.SYSTEMS))
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_system_exact_integer_bit_identical(an5d, name, dtype):
    ndim, rad, shape, nf, _ = inputs.system_problem(name)
    tab = inputs.system_table(ndim, rad, shape, nf, seed=77, kind="pm1")
    f = inputs.system_fields(555, nf, EXT, kind="pm")
    taps = nf * ((2 * rad + 1) ** ndim if shape == inputs.BOX else 2 * ndim * rad + 1)
    lim = 2.0 ** (24 if dtype == torch.float32 else 53)
    st = an5d.System(ndim, rad, shape, tab, dtype)
    for cfg in configs(an5d, st, EXT):
        T, bound = 0, 1.0
        while T < 2 * cfg["bT"] + 3 and bound * taps < lim:
            bound *= taps
            T += 1
        got, _ = run_system(an5d, ndim, rad, shape, tab, f, T, dtype, cfg)
        assert np.array_equal(got, oracle.run_system(f, rad, shape, tab, T, NP[dtype])), (name, cfg, T)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_decoupled_system_equals_single_field_runs(an5d, dtype):
    ndim, rad, shape, nf, tab = inputs.system_problem("star2d1r-x2")
    tab = tab.copy()
    tab[0, 1] = 0
    tab[1, 0] = 0
    f = inputs.system_fields(21, nf, EXT)
    st = an5d.System(ndim, rad, shape, tab, dtype)
    s1s = [an5d.Stencil(ndim, rad, shape, tab[i, i], 1.0, dtype) for i in range(nf)]
    n_checked = 0
    for cfg in configs(an5d, st, EXT):
        try:   # the single-field build may lack this (b_T, vec)
            s1s[0].describe(EXT, cfg)
        except an5d.AN5DError:
            continue
        n_checked += 1
        got, _ = run_system(an5d, ndim, rad, shape, tab, f, 9, dtype, cfg)
        for i in range(nf):
            s1 = s1s[i]
            a = an5d.to_grid(torch.from_numpy(f[i].astype(NP[dtype])).cuda(), rad)
            b = an5d.empty_grid(EXT, rad, dtype)
            s1.run(a, b, 9, cfg)
            torch.cuda.synchronize()
            assert np.array_equal(got[i], b.cpu().numpy()), (cfg, i)
    assert n_checked > 0


@pytest.mark.parametrize("name", sorted(inputs.SYSTEMS))
def test_system_write_count_map(an5d, name):
    ndim, rad, shape, nf, tab = inputs.system_problem(name)
    st = an5d.System(ndim, rad, shape, tab, torch.float32)
    f = inputs.system_fields(5, nf, EXT)
    a = an5d.to_fields(torch.from_numpy(f.astype(np.float32)).cuda(), rad)
    b = an5d.empty_fields(nf, EXT, rad, torch.float32)
    for cfg in configs(an5d, st, EXT):
        wc = torch.zeros((nf,) + EXT, dtype=torch.int32, device="cuda")
        st.copy_ring(a, b)
        st.sweep(a, b, cfg["bT"], cfg, write_count=wc)
        torch.cuda.synchronize()
        w = wc.cpu().numpy()
        core = (slice(None), slice(rad, EXT[0] - rad), slice(rad, EXT[1] - rad))
        assert np.all(w[core] == 1), cfg
        w[core] = 0
        assert not w.any(), cfg


@pytest.mark.parametrize("name", sorted(inputs.SYSTEMS))
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_system_full_T_planner_config(an5d, name, dtype):
    ndim, rad, shape, nf, tab = inputs.system_problem(name)
    ext = (2048 + 2 * rad,) * 2
    st = an5d.System(ndim, rad, shape, tab, dtype)
    pick = st.plan_config((16384 + 2 * rad,) * 2, 1000)
    cfg = st.plan_config(ext, 1000, {"bT": pick["bT"], "vec": pick["vec"]})
    f = inputs.system_fields(inputs.DEFAULT_SEED, nf, ext)
    got, _ = run_system(an5d, ndim, rad, shape, tab, f, 1000, dtype, cfg)
    exp = oracle.run_system(f, rad, shape, tab, 1000, NP[dtype])
    assert rings_equal(got, exp, rad), cfg
    assert rel_linf(got, exp, rad) <= TOL[dtype], (name, cfg, rel_linf(got, exp, rad))
