"""Host-side logic without a GPU: C-ABI exports, bit-exact bookkeeping, schedule, FLOP accounting."""
import json
import math
import os
import re

import pytest

import oracle.geometry as og

GOLD = os.path.join(os.path.dirname(__file__), "golden")
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_library_loads_and_exports_every_declared_symbol(an5d):
    """Every function declared in include/an5d.h is exported by libAN5D.so."""
    import ctypes
    hdr = open(os.path.join(REPO, "include", "an5d.h")).read()
    declared = set(re.findall(r"^\s*(?:an5d_status|const char\*|int64_t)\s+(an5d_\w+)\s*\(", hdr, re.M))
    assert {"an5d_create", "an5d_run", "an5d_destroy", "an5d_sweep", "an5d_describe"} <= declared
    lib = ctypes.CDLL(an5d.LIB_PATH)
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert set(an5d.EXPORTED_SYMBOLS) == declared
    assert "sm_100a" in an5d.version()


def test_oracle_geometry_spec_examples():
    """The paper's formulas (oracle.geometry) reproduce SPEC.md's worked examples."""
    ex = _gold("spec_geometry.json")["examples"]
    e = ex[0]
    assert og.n_thr(e["bS"]) == e["n_thr"]
    assert [og.compute_region(b, e["bT"], e["rad"]) for b in e["bS"]] == e["compute_region"]
    ntb = og.n_tb(e["I_S"][1:], e["bS"], e["bT"], e["rad"])
    assert ntb == e["n_tb"]
    assert og.n_tb_prime(e["I_S"][0], e["h_SN"], ntb) == e["n_tb_prime"]
    assert og.stream_overlap(e["bT"], e["rad"]) == e["stream_overlap"]
    e = ex[1]
    assert og.compute_region(e["bS"][0], e["bT"], e["rad"]) == e["compute_region"][0]
    assert og.n_tb(e["I_S"], e["bS"], e["bT"], e["rad"]) == e["n_tb"]
    e = ex[2]
    assert og.compute_region(e["bS"][0], e["bT"], e["rad"]) < 1


def test_stream_overlap_closed_form():
    """2 sum_{T<bT} rad (bT - T) == rad bT (bT + 1)."""
    for bT in range(1, 17):
        for rad in range(1, 5):
            assert og.stream_overlap(bT, rad) == rad * bT * (bT + 1)


def test_valid_region_recurrence():
    for bS in (16, 64, 256):
        for rad in (1, 2):
            for T in range(0, 5):
                assert og.valid_region(bS, T + 1, rad) == og.valid_region(bS, T, rad) - 2 * rad


def test_valid_region_brute_force_dependency_cone():
    """P:336 'the size of the region with valid computation ... b_S - 2 T rad': brute force on
    position SETS (no formula) -- a cell is valid at level T when all its stencil inputs were valid
    at level T-1, starting from the whole loaded tile at T = 0 -- gives exactly the cells
    [T rad, b_S - T rad), and the compute region is the level-b_T set."""
    for bS in (7, 16, 33, 64):
        for rad in (1, 2, 3, 4):
            valid = set(range(bS))
            for T in range(1, 9):
                valid = {x for x in valid if all(x + d in valid for d in range(-rad, rad + 1))}
                w = og.valid_region(bS, T, rad)
                assert len(valid) == max(0, w), (bS, rad, T)
                if w > 0:
                    assert valid == set(range(T * rad, bS - T * rad))
                    assert og.compute_region(bS, T, rad) == len(valid)


def test_paper_adjustment_condition_literal_values():
    """The printed final-block condition '(I_T mod b_T) != 0 or ((I_T / b_T) mod 2) !=
    (b_T mod 2)', evaluated by hand for a few cases (integer division I_T / b_T):
      (1000, 4): 0, 250 mod 2 = 0 == 4 mod 2 = 0            -> False
      (1000, 3): 1000 mod 3 = 1                             -> True
      (12, 3):   0, 4 mod 2 = 0 != 3 mod 2 = 1              -> True  (fires with an even sweep
                 count and odd b_T, where reading R-7 needs no fix: SURVEY C-7)
      (9, 3):    0, 3 mod 2 = 1 == 1                        -> False
      (10, 10):  0, 1 mod 2 = 1 != 10 mod 2 = 0             -> True
      (16, 8):   0, 2 mod 2 = 0 == 0                        -> False
      (7, 2):    7 mod 2 = 1                                -> True"""
    cases = {(1000, 4): False, (1000, 3): True, (12, 3): True, (9, 3): False, (10, 10): True, (16, 8): False,
             (7, 2): True}
    for (IT, bT), want in cases.items():
        assert og.paper_adjustment_condition(IT, bT) is want, (IT, bT)


@pytest.mark.parametrize("case", _gold("schedule_survey.json")["cases"])
def test_schedule_matches_survey_table(case, an5d):
    """Library (C++) and oracle (Python) schedules equal SURVEY's independently computed table."""
    exp = [d for d, n in case["degrees"] for _ in range(n)]
    deg, copy = og.schedule(case["T"], case["bT"])
    assert deg == exp and copy == case["copy"]
    deg2, copy2 = an5d.schedule(case["T"], case["bT"])
    assert deg2 == exp and copy2 == case["copy"]


def test_schedule_invariants(an5d):
    for T in range(0, 60):
        for bT in range(1, 11):
            deg, copy = an5d.schedule(T, bT)
            assert (deg, copy) == og.schedule(T, bT)
            assert sum(deg) == T
            assert all(1 <= d <= bT for d in deg)
            if T > 0:
                assert (len(deg) % 2 == 1) or copy
                assert not (copy and len(deg) % 2 == 1)
            # the paper's literal condition never misses a case that needs adjusting
            if T % bT != 0:
                assert og.paper_adjustment_condition(T, bT)


@pytest.mark.parametrize("name", ["star2d1r", "box2d2r", "j2d5pt", "star3d1r", "box3d1r", "star3d4r", "j3d27pt",
                                  "box2d4r", "star2d4r"])
@pytest.mark.parametrize("dtype_name", ["float32", "float64"])
def test_describe_matches_paper_formulas(name, dtype_name, an5d):
    """an5d_describe (C++) is bit-exact with the paper's formulas (oracle.geometry) for every
    configuration the library exposes."""
    import torch

    import inputs
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    dtype = getattr(torch, dtype_name)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    ext = [16384 + 2 * rad] * 2 if ndim == 2 else [512 + 2 * rad] * 3
    n = 0
    for bT in range(1, 11):
        for vec in (1, 2, 4, 8):
            for h in (128, 500, 4096):
                try:
                    g = st.describe(ext, {"bT": bT, "vec": vec, "h": h})
                except an5d.AN5DError as e:
                    assert e.status in (2, 5)   # infeasible / no instance
                    continue
                n += 1
                nb = ndim - 1
                I_S = [e - 2 * rad for e in ext]
                bS = g["bS"][:nb]
                assert g["compute"][:nb] == [og.compute_region(b, bT, rad) for b in bS]
                assert g["n_tiles"][:nb] == [math.ceil(I / c) for I, c in zip(I_S[1:], g["compute"][:nb])]
                assert g["n_tb"] == og.n_tb(I_S[1:], bS, bT, rad)
                assert g["n_tb_prime"] == og.n_tb_prime(I_S[0], g["h"], g["n_tb"])
                assert g["stream_overlap"] == og.stream_overlap(bT, rad)
                assert all(hl >= bT * rad for hl in g["halo_loaded"][:nb])
                assert all(bl == c + 2 * hl for bl, c, hl in zip(g["bS_loaded"][:nb], g["compute"][:nb],
                                                                  g["halo_loaded"][:nb]))
    assert n > 0


def test_create_rejects_bad_arguments(an5d):
    import numpy as np
    import torch
    with pytest.raises(an5d.AN5DError) as e:
        an5d.Stencil(2, 1, an5d.STAR, np.ones((3, 3)), 1.0, torch.float32)   # off-axis non-zero
    assert e.value.status == 4
    with pytest.raises(an5d.AN5DError) as e:
        an5d.Stencil(2, 5, an5d.BOX, np.ones((11, 11)), 1.0, torch.float32)
    assert e.value.status == 1
    with pytest.raises(an5d.AN5DError) as e:
        an5d.Stencil(4, 1, an5d.BOX, np.ones((3, 3, 3, 3)), 1.0, torch.float32)
    assert e.value.status == 1
    with pytest.raises(an5d.AN5DError) as e:
        an5d.Stencil(2, 1, an5d.BOX, np.ones((3, 3)), 0.0, torch.float32)
    assert e.value.status == 1
    # gradient2d (Table 2): 2D radius 1 only, only the centre entry may be non-zero
    with pytest.raises(an5d.AN5DError) as e:
        an5d.Stencil(2, 2, an5d.GRAD, np.zeros((5, 5)), 1.0, torch.float32)
    assert e.value.status == 5
    off = np.zeros((3, 3))
    off[0, 1] = 0.5
    with pytest.raises(an5d.AN5DError) as e:
        an5d.Stencil(2, 1, an5d.GRAD, off, 1.0, torch.float32)
    assert e.value.status == 4
    cen = np.zeros((3, 3))
    cen[1, 1] = 0.5
    for c0 in (0.0, -1.0, 1e-39, float("inf")):   # c_0 must be a normal number (branch-free 1/sqrt)
        with pytest.raises(an5d.AN5DError) as e:
            an5d.Stencil(2, 1, an5d.GRAD, cen, c0, torch.float32)
        assert e.value.status in (1, 5), c0
    an5d.Stencil(2, 1, an5d.GRAD, cen, 1.0, torch.float32)


def test_create_system_rejects_bad_arguments(an5d):
    """an5d_create_system (multi-field systems, NEXT N4): block count, STAR off-axis entries in any
    block, 3D with several fields, field count -- all rejected before anything runs."""
    import numpy as np
    import torch
    import inputs
    tab = inputs.system_table(2, 1, inputs.STAR, 2, seed=1)
    an5d.System(2, 1, inputs.STAR, tab, torch.float32)
    with pytest.raises(ValueError):
        an5d.System(2, 1, inputs.STAR, tab[:1], torch.float32)           # not (n_f, n_f, ...)
    bad = tab.copy()
    bad[1, 0, 0, 0] = 0.25                                               # STAR off-axis, block (1, 0)
    with pytest.raises(an5d.AN5DError) as e:
        an5d.System(2, 1, inputs.STAR, bad, torch.float32)
    assert e.value.status == 4
    t3 = np.zeros((2, 2, 3, 3, 3))
    with pytest.raises(an5d.AN5DError) as e:
        an5d.System(3, 1, inputs.BOX, t3, torch.float32)
    assert e.value.status == 5
    with pytest.raises(an5d.AN5DError) as e:
        an5d.System(2, 1, inputs.BOX, np.zeros((9, 9, 3, 3)), torch.float32)
    assert e.value.status == 1


def test_set_comm_argument_errors(an5d):
    """an5d_set_comm: bad rank / nranks are rejected before NCCL is touched; detaching a plan that
    has no communicator is a no-op."""
    import numpy as np
    import torch
    import inputs
    ndim, rad, shape, tab, div = inputs.benchmark_problem("star2d1r")
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    st.set_comm(None)
    for rank, nranks in ((0, 0), (2, 2), (-1, 2)):
        with pytest.raises(an5d.AN5DError) as e:
            st.set_comm(b"\0" * 128, rank, nranks, 100, 0, 2)
        assert e.value.status == 1


def test_flops_per_cell_table2():
    from paper_2001_01473_b200 import perf
    import inputs
    g = _gold("table2_flops.json")["flops"]
    for name, (ndim, rad, shape, has_div) in inputs.BENCHMARKS.items():
        assert perf.flops_per_cell(ndim, rad, shape, has_div) == g[name], name
    # eff_ALU for star2d1r: 4 FMA + 1 MUL -> 9/10
    assert abs(perf.eff_alu(2, 1, 0, False) - 0.9) < 1e-15


def test_direct_variant_config(an5d):
    """Partial sums off (config field `direct`, Table 1 "Otherwise" P:262-270): 2D box instances
    exist and describe like the associative ones (same geometry formulas); 3D or an out-of-range
    value is rejected before any launch."""
    import torch

    import inputs
    ndim, rad, shape, tab, div = inputs.benchmark_problem("box2d2r")
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    ext = [16384 + 2 * rad] * 2
    for bT in (1, 2):   # the default build has box2d2r b_T 1..2 (build.py CORE)
        g0 = st.describe(ext, {"bT": bT, "vec": 8, "h": 256})
        g1 = st.describe(ext, {"bT": bT, "vec": 8, "h": 256, "direct": 1})
        for k in ("bS", "compute", "halo_loaded", "n_tiles", "n_tb", "n_tb_prime", "stream_overlap"):
            assert g0[k] == g1[k], k
    with pytest.raises(an5d.AN5DError) as e:
        st.describe(ext, {"bT": 2, "vec": 8, "h": 256, "direct": 2})
    assert e.value.status == 1
    ndim, rad, shape, tab, div = inputs.benchmark_problem("box3d1r")
    st3 = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    with pytest.raises(an5d.AN5DError) as e:
        st3.describe([66, 66, 66], {"bT": 1, "vec": 2, "h": 32, "direct": 1})
    assert e.value.status == 5


def test_run_table_unit_count(an5d, monkeypatch):
    """2D run schedule: with AN5D_RUN_FRAC=0 every unit is one stream block
    (n_units == n_tb_prime); with runs, fewer units, never fewer than one per tile, and a
    smaller table when it is shaped for fewer warps (longer runs); the same for 3D."""
    import torch

    import inputs
    ndim, rad, shape, tab, div = inputs.benchmark_problem("star2d1r")
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    ext = [16384 + 2 * rad] * 2
    cfg = {"bT": 4, "vec": 8, "h": 64}
    monkeypatch.setenv("AN5D_RUN_FRAC", "0")
    g0 = st.describe(ext, cfg)
    assert g0["n_units"] == g0["n_tb_prime"]
    monkeypatch.delenv("AN5D_RUN_FRAC")
    g1 = st.describe(ext, cfg)
    assert g0["n_tiles"][0] <= g1["n_units"] < g0["n_tb_prime"]
    monkeypatch.setenv("AN5D_RUN_WARPS", "64")
    g2 = st.describe(ext, cfg)
    assert g0["n_tiles"][0] <= g2["n_units"] <= g1["n_units"]
    monkeypatch.delenv("AN5D_RUN_WARPS")
    s3 = an5d.Stencil(3, 1, shape, *inputs.coeff_table(3, 1, shape, seed=4), torch.float32)
    g3 = s3.describe([514] * 3, {"bT": 2, "h": 16, "vec": 2})
    assert g3["n_tb"] <= g3["n_units"] < g3["n_tb_prime"]
    monkeypatch.setenv("AN5D_RUN_FRAC", "0")
    g4 = s3.describe([514] * 3, {"bT": 2, "h": 16, "vec": 2})
    assert g4["n_units"] == g4["n_tb_prime"] == g3["n_tb_prime"]


@pytest.mark.parametrize("name", ["star3d1r", "star3d2r", "box3d1r", "box3d2r", "j3d27pt"])
@pytest.mark.parametrize("dtype_name", ["float32", "float64"])
def test_3d_x_halo_rule(name, dtype_name, an5d):
    """Loaded x halo of the 3D layouts without x staging (x-pair tiles): fp32 with
    b_T rad = 2 (mod 4) loads exactly b_T rad (compute width 64 - 2 b_T rad); every other case
    rounds b_T rad up to a 16-byte vector (4 fp32 / 2 fp64 cells).  The compute region and tile
    count then follow P:320 / P:323 from the logical b_S the library reports."""
    import torch

    import inputs
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    dtype = getattr(torch, dtype_name)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    ext = [512 + 2 * rad] * 3
    A = 4 if dtype == torch.float32 else 2
    n = 0
    for bT in range(1, 7):
        try:
            g = st.describe(ext, {"bT": bT, "vec": 2, "h": 64, "n_thr": 256, "bS": [32, 0]})
        except an5d.AN5DError as e:
            assert e.status in (2, 5)
            continue
        n += 1
        hr = bT * rad
        want = hr if (A == 4 and hr % 4 == 2) else -(-hr // A) * A
        assert g["bS_loaded"][1] == 64 and g["halo_loaded"][1] == want, (bT, g)
        assert g["compute"][1] == 64 - 2 * want == og.compute_region(g["bS"][1], bT, rad), (bT, g)
        assert g["n_tiles"][1] == math.ceil(512 / g["compute"][1]), (bT, g)
    assert n > 0
