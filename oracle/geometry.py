"""Blocking bookkeeping written out from the paper -- TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Every function restates one formula of PAPER.md section 4 in the paper's notation, so the
library's C++ (an5d_describe / an5d_schedule) can be compared with it bit-exactly.
"""
from __future__ import annotations

import math


def n_thr(bS):
    """n_thr = prod_{i=1}^{N-1} b_S_i  (one cell per thread in the paper)."""
    return math.prod(bS)


def compute_region(bS_i: int, bT: int, rad: int) -> int:
    """Threads per dimension that store results: b_S_i - 2 * b_T * rad."""
    return bS_i - 2 * bT * rad


def valid_region(bS_i: int, T: int, rad: int) -> int:
    """Width of the valid computation at time-step T: b_S_i - 2 * T * rad."""
    return bS_i - 2 * T * rad


def n_tb(I_S, bS, bT: int, rad: int) -> int:
    """n_tb = prod ceil(I_S_i / (b_S_i - 2 b_T rad))."""
    return math.prod(-(-I // compute_region(b, bT, rad)) for I, b in zip(I_S, bS))


def n_tb_prime(I_SN: int, h_SN: int, ntb: int) -> int:
    """n'_tb = ceil(I_SN / h_SN) * n_tb."""
    return -(-I_SN // h_SN) * ntb


def stream_overlap(bT: int, rad: int) -> int:
    """Redundant sub-planes between consecutive stream blocks: 2 * sum_{T=0}^{b_T-1} rad (b_T - T)
    (P:427), evaluated literally (the closed form rad b_T (b_T+1) is checked in the tests)."""
    return 2 * sum(rad * (bT - T) for T in range(0, bT))


def schedule(I_T: int, bT: int):
    """Sweep degrees of the host loop under DESIGN.md reading R-7 (SURVEY C-7).

    Each kernel call advances b_T steps; the final block is reduced so the total is I_T, and the
    result must be in grid_out, i.e. the number of buffer flips (sweeps) must be odd: if it is
    even, the last sweep of degree >= 2 is split into (ceil(d/2), floor(d/2)); if all degrees are
    1, a trailing interior copy is appended.  Returns (degrees, trailing_copy).
    """
    if I_T <= 0:
        return [], False
    deg = [bT] * (I_T // bT)
    if I_T % bT:
        deg.append(I_T % bT)
    if len(deg) % 2 == 0:
        for i in range(len(deg) - 1, -1, -1):
            if deg[i] >= 2:
                d = deg[i]
                deg[i:i + 1] = [(d + 1) // 2, d // 2]
                return deg, False
        return deg, True
    return deg, False


def paper_adjustment_condition(I_T: int, bT: int) -> bool:
    """The paper's literal final-block condition:
    (I_T mod b_T) != 0  or  ((I_T / b_T) mod 2) != (b_T mod 2)."""
    return (I_T % bT) != 0 or ((I_T // bT) % 2) != (bT % 2)
