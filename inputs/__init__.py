"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module is deliberately separate from both ``oracle/`` and the product package
``paper_2001_01473_b200``: it holds *no* stencil arithmetic, only

* a counter-based hash (murmur3 ``fmix32`` chained over seed and cell index), so every
  cell value is a pure function of (seed, global linear index) and any sub-block or
  GPU decomposition sees identical values (SURVEY.md §8(d) "Values" column);
* grid / coefficient-table generators built on it;
* the benchmark catalogue of PAPER.md Table 2: name -> (ndim, rad, shape,
  divisor?).  This is *structure* of the paper's workloads (which taps exist), not the
  update formula.

Recipe:
  value(seed, i)  = (fmix32(fmix32(fmix32(lo(seed) ^ 0x9E3779B9) ^ hi(seed) ^ hi(i)) ^ lo(i)) >> 8) / 2^24
  i.e. a 24-bit uniform in [0, 1): exactly representable in fp32 and fp64, never denormal.
  Dyadic coefficient tables: random integer weights m_d in [1, 1024] for every tap of the
  shape, the centre weight raised so that sum(m_d) = 2^p, c_d = m_d / 2^p  -> sum c_d == 1
  exactly in both precisions.
  j-stencils (divisor): integer taps m_d in [1, 1024], divisor = sum(m_d).
"""
from __future__ import annotations

import itertools
import numpy as np

M32 = 0xFFFFFFFF
DEFAULT_SEED = 0x200101473

STAR, BOX, GRAD = 0, 1, 2

# PAPER.md Table 2: stencil name -> (ndim, rad, shape, has_divisor)
# j2d5pt = star2d1r taps / c0; j2d9pt = star2d2r taps / c0 ("2nd-order" P:641-642);
# j3d27pt = box3d1r taps / c0; j2d9pt-gol = box2d1r taps / c0.
BENCHMARKS = {}
for _r in range(1, 5):
    BENCHMARKS[f"star2d{_r}r"] = (2, _r, STAR, False)
    BENCHMARKS[f"box2d{_r}r"] = (2, _r, BOX, False)
    BENCHMARKS[f"star3d{_r}r"] = (3, _r, STAR, False)
    BENCHMARKS[f"box3d{_r}r"] = (3, _r, BOX, False)
BENCHMARKS["j2d5pt"] = (2, 1, STAR, True)
BENCHMARKS["j2d9pt"] = (2, 2, STAR, True)
BENCHMARKS["j3d27pt"] = (3, 1, BOX, True)
# j2d9pt-gol = box2d1r taps / c0 (Table 2, the "game of life"-shaped 9-point Jacobi)
BENCHMARKS["j2d9pt-gol"] = (2, 1, BOX, True)
# gradient2d (Table 2): non-linear; "divisor" slot = c_0 under the square root
BENCHMARKS["gradient2d"] = (2, 1, GRAD, True)


def _fmix32(h):
    """murmur3 finaliser on uint64 arrays holding 32-bit values (numpy)."""
    h = h & M32
    h ^= h >> np.uint64(16)
    h = (h * np.uint64(0x85EBCA6B)) & M32
    h ^= h >> np.uint64(13)
    h = (h * np.uint64(0xC2B2AE35)) & M32
    h ^= h >> np.uint64(16)
    return h


def hash32(seed: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based 32-bit hash of (seed, idx) for an array of non-negative int64 indices."""
    idx = np.asarray(idx, dtype=np.uint64)
    k = _fmix32(np.uint64((seed & M32) ^ 0x9E3779B9))
    k = _fmix32(k ^ np.uint64((seed >> 32) & M32) ^ (idx >> np.uint64(32)))
    return _fmix32(k ^ (idx & np.uint64(M32)))


def uniform24(seed: int, idx: np.ndarray) -> np.ndarray:
    """24-bit uniform values in [0, 1) as float64 (exact in fp32 too)."""
    return (hash32(seed, idx) >> np.uint64(8)).astype(np.float64) * (1.0 / (1 << 24))


def small_int(seed: int, idx: np.ndarray, n: int) -> np.ndarray:
    """Integers in [0, n) (exact-integer mode inputs)."""
    return (hash32(seed, idx) % np.uint64(n)).astype(np.float64)


def global_grid(seed: int, extents, outer_offset: int = 0, outer_count: int | None = None,
                global_extents=None, kind: str = "uniform", n_int: int = 16) -> np.ndarray:
    """Dense float64 array of cell values for the array ``extents`` (ring included).

    With ``global_extents`` / ``outer_offset`` the block is the planes
    [outer_offset, outer_offset + outer_count) of a larger global array, and each cell's
    value is keyed by its *global* linear index, so any slab decomposition sees the same
    values.
    """
    extents = tuple(int(e) for e in extents)
    g_ext = tuple(int(e) for e in (global_extents or extents))
    if outer_count is None:
        outer_count = extents[0]
    inner = int(np.prod(g_ext[1:]))
    base = np.arange(outer_count, dtype=np.int64)[:, None] + outer_offset
    lin = (base * inner + np.arange(inner, dtype=np.int64)[None, :]).reshape(-1)
    if kind == "uniform":
        v = uniform24(seed, lin)
    elif kind == "int":
        v = small_int(seed, lin, n_int)
    elif kind == "pm":
        v = small_int(seed, lin, 3) - 1.0
    else:
        raise ValueError(kind)
    return v.reshape((outer_count,) + g_ext[1:])


def tap_offsets(ndim: int, rad: int, shape: int):
    """Offsets (outer..x order) of the taps that exist for a shape, lexicographic order.

    star: centre plus +-k along one axis at a time (Table 2 star rows);
    box: the full (2r+1)^N cube (Table 2 box rows).
    """
    offs = []
    for d in itertools.product(range(-rad, rad + 1), repeat=ndim):
        nz = sum(1 for v in d if v != 0)
        if shape == BOX or nz <= 1:
            offs.append(d)
    return offs


def coeff_table(ndim: int, rad: int, shape: int, seed: int, kind: str = "dyadic",
                symmetric: bool = False):
    """Dense (2r+1)^ndim float64 coefficient table (index order outer..x) and divisor.

    kind='dyadic': sum == 1 exactly (C-2); kind='int': integer taps, divisor = sum (j-stencils);
    kind='small': distinct small integers 1..n_taps, divisor 1 (exact-integer mode);
    kind='pm1': random +-1 per tap, divisor 1 (exact-integer mode with slow growth).
    ``symmetric`` makes c_d == c_{-d} (linear-field pin).
    """
    w = 2 * rad + 1
    tab = np.zeros((w,) * ndim, dtype=np.float64)
    offs = tap_offsets(ndim, rad, shape)
    for n, d in enumerate(offs):
        key = d
        if symmetric:
            neg = tuple(-v for v in d)
            key = max(d, neg)  # canonical representative of the +-d pair
        lin = 0
        for v in key:
            lin = lin * w + (v + rad)
        if kind == "small":
            m = float(n + 1)
        elif kind == "pm1":
            m = 1.0 if int(hash32(seed + 1, np.array([lin]))[0]) & 1 else -1.0
        else:
            m = float(1 + int(hash32(seed + 1, np.array([lin]))[0] % np.uint64(1024)))
        tab[tuple(v + rad for v in d)] = m
    divisor = 1.0
    if kind == "dyadic":
        s_other = tab.sum() - tab[tuple(rad for _ in range(ndim))]
        p = 0
        while (1 << p) <= s_other:
            p += 1
        tab[tuple(rad for _ in range(ndim))] = float((1 << p) - s_other)
        tab /= float(1 << p)
    elif kind == "int":
        divisor = float(tab.sum())
    elif kind not in ("small", "pm1"):
        raise ValueError(kind)
    return tab, divisor


# Multi-field systems (NEXT N4, "multi-output temporal blocking ... multi-statement
# stencils"): name -> (ndim, rad, shape, n_fields).  n_f arrays updated together, statement i
# reading the previous step of every array through a Table-2-shaped block (i, j).
SYSTEMS = {
    "star2d1r-x2": (2, 1, STAR, 2),
    "box2d1r-x2": (2, 1, BOX, 2),
}


def system_table(ndim: int, rad: int, shape: int, nf: int, seed: int, kind: str = "dyadic"):
    """(n_f, n_f, (2r+1,)*ndim) float64 block table; block [i, j] = field j's contribution to field i.

    kind='dyadic': integer weights m in [1, 1024] on every tap of every block, the diagonal block's
    centre raised so that each OUTPUT field's weights sum to 2^p, divided by 2^p: every statement
    sums to 1 exactly (a constant state is a fixed point; values stay in [0, 1]).
    kind='pm1': +-1 per tap (exact-integer mode)."""
    w = 2 * rad + 1
    tab = np.zeros((nf, nf) + (w,) * ndim, dtype=np.float64)
    offs = tap_offsets(ndim, rad, shape)
    centre = tuple(rad for _ in range(ndim))
    for i in range(nf):
        for j in range(nf):
            for d in offs:
                lin = ((i * nf + j) * w ** ndim + sum((v + rad) * w ** (ndim - 1 - a) for a, v in enumerate(d)))
                h = int(hash32(seed + 3, np.array([lin]))[0])
                if kind == "pm1":
                    m = 1.0 if h & 1 else -1.0
                else:
                    m = float(1 + h % 1024)
                tab[(i, j) + tuple(v + rad for v in d)] = m
        if kind == "dyadic":
            s_other = tab[i].sum() - tab[(i, i) + centre]
            p = 0
            while (1 << p) <= s_other:
                p += 1
            tab[(i, i) + centre] = float((1 << p) - s_other)
            tab[i] /= float(1 << p)
        elif kind != "pm1":
            raise ValueError(kind)
    return tab


def system_problem(name: str, seed: int = DEFAULT_SEED):
    """(ndim, rad, shape, n_fields, block table) of a catalogued multi-field system."""
    ndim, rad, shape, nf = SYSTEMS[name]
    return ndim, rad, shape, nf, system_table(ndim, rad, shape, nf, seed)


def system_fields(seed: int, nf: int, extents, kind: str = "uniform") -> np.ndarray:
    """(n_f, *extents) float64 seeded fields: field f uses seed + 0x1000 * f."""
    return np.stack([global_grid(seed + 0x1000 * f, extents, kind=kind) for f in range(nf)])


def gradient_params(seed: int):
    """gradient2d constants (Table 2 P:698-699 leaves them open): centre c = m / 1024 with
    m in [256, 768) and c_0 = 1 + m' / 1024 with m' in [0, 1024) -- dyadic (exact in fp32 and
    fp64).  |c| < 1 and c_0 >= 1 keep a T-step run bounded: f stays in [0, (max f_0) + 1/(1-c)]."""
    h = hash32(seed + 2, np.array([0, 1]))
    return 0.25 + float(int(h[0]) % 512) / 1024.0, 1.0 + float(int(h[1]) % 1024) / 1024.0


def benchmark_problem(name: str, seed: int = DEFAULT_SEED):
    """(ndim, rad, shape, coeff_table, divisor) for a Table-2 benchmark with seeded coefficients.
    gradient2d: a 3x3 table holding only the centre c, and c_0 in the divisor slot."""
    ndim, rad, shape, has_div = BENCHMARKS[name]
    if shape == GRAD:
        c, c0 = gradient_params(seed)
        tab = np.zeros((3, 3))
        tab[1, 1] = c
        return ndim, rad, shape, tab, c0
    tab, div = coeff_table(ndim, rad, shape, seed, kind="int" if has_div else "dyadic")
    return ndim, rad, shape, tab, div


def uniform24_torch(seed: int, lin):
    """Same generator as :func:`uniform24` on a torch int64 tensor of indices (any device).

    Plumbing for large bench grids (input generation on the GPU); bit-identical to the
    numpy version (tests check it).
    """
    import torch

    def fmix(h):
        h = h & M32
        h = h ^ (h >> 16)
        h = (h * 0x85EBCA6B) & M32
        h = h ^ (h >> 13)
        h = (h * 0xC2B2AE35) & M32
        h = h ^ (h >> 16)
        return h

    k0 = int(_fmix32(np.uint64((seed & M32) ^ 0x9E3779B9)))
    hi = (lin >> 32) & M32
    k = fmix(hi ^ (k0 ^ ((seed >> 32) & M32)))
    h = fmix(k ^ (lin & M32))
    return (h >> 8).to(torch.float64) * (1.0 / (1 << 24))
