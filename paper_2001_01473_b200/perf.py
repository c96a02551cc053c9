"""Performance accounting used by bench.py: FLOP/cell, eff_ALU and the b_T-adjusted roofline.

Pure host arithmetic on counts (no cell data).  Citations:
  * FLOP/cell: PAPER.md Table 2, with the FMA-merging rule of P:589-605 (k products ->
    k-1 FMA + 1 MUL; the j-stencil division becomes one MUL under fast math).
  * eff_ALU: P:611-614.
  * roofline: BASELINE.json metric "min(FMA peak, HBM BW x bT / bytes-per-cell-per-step),
    accounting for halo redundancy", written out in SURVEY.md §8(d).
"""
from __future__ import annotations

STAR, BOX, GRAD = 0, 1, 2


def n_taps(ndim: int, rad: int, shape: int) -> int:
    return (2 * rad + 1) ** ndim if shape == BOX else 2 * ndim * rad + 1


def flops_per_cell(ndim: int, rad: int, shape: int, has_div: bool, nf: int = 1) -> int:
    """Table 2: k products summed = k FMA-equivalent ops counted as 2k-1 FLOPs, +1 for /c_0;
    gradient2d: the printed 19.  Multi-field systems (nf > 1): per cell of one field,
    its statement sums nf x taps products (2 nf taps - 1 FLOPs)."""
    if shape == GRAD:
        return 19
    return 2 * nf * n_taps(ndim, rad, shape) - 1 + (1 if has_div else 0)


def op_mix(ndim: int, rad: int, shape: int, has_div: bool, nf: int = 1):
    """(n_FMA, n_MUL, n_ADD + n_OTHER) per cell under the paper's mapping.
    gradient2d: 2 FMA (a square added to a square), 3 MUL (two squares, c f),
    4 differences + 3 adds, and sqrt + division counted as OTHER (R-17)."""
    if shape == GRAD:
        return 2, 3, 9
    k = nf * n_taps(ndim, rad, shape)
    return k - 1, 1 + (1 if has_div else 0), 0


def eff_alu(ndim: int, rad: int, shape: int, has_div: bool, nf: int = 1) -> float:
    """eff_ALU = (2 FMA + MUL + ADD + OTHER) / (2 (FMA + MUL + ADD + OTHER))."""
    f, m, a = op_mix(ndim, rad, shape, has_div, nf)
    return (2 * f + m + a) / (2 * (f + m + a))


def fp_peak_flops(dtype_bytes: int, n_sm: int = 148, clock_mhz: float = 1965.0) -> float:
    """CUDA-core FMA peak (FLOP/s) from unit counts and clock:
    B200 SM = 4 SMSPs x 32 FP32 lanes = 128 FFMA/clk; 64 FP64 lanes (DFMA) per SM."""
    lanes = 128 if dtype_bytes == 4 else 64
    return n_sm * lanes * 2.0 * clock_mhz * 1e6


def roofline(*, ndim, rad, shape, has_div, dtype_bytes, bT, tile_loaded, tile_compute, h, hbm_gbs,
             fp_peak, nf=1):
    """b_T-adjusted roofline in cells/s for a configuration.

    With the logical tile b_i = C_i + 2 b_T rad (the paper's b_S incl. halo), compute
    region C_i and stream block h:
      R_read = (prod b / prod C) * (h + 2 b_T rad) / h                  halo + stream-overlap reloads
      R_comp = (1/b_T) sum_{T=1..b_T} (prod (b_i - 2 T rad) / prod C) * (h + 2 rad (b_T - T)) / h
               (level T only has to compute its shrinking valid region)
      roof   = min(P eff_ALU / (F R_comp), B b_T / (n_w (R_read + 1)))
      ideal  = min(P eff_ALU / F, B b_T / (2 n_w))                      (R = 1)
    Only useful work is credited: algorithmic bytes per cell-step n_w (R_read + 1) / b_T and FLOPs
    per cell-step F R_comp.  The kernel's actual redundancy (its loaded window is the logical tile
    rounded up to whole 16-byte vectors, and it computes that whole window at every level) is
    reported separately as R_read_kernel / R_comp_kernel.
    """
    import math
    F = flops_per_cell(ndim, rad, shape, has_div, nf)      # per cell of one field (nf: systems)
    eff = eff_alu(ndim, rad, shape, has_div, nf)
    C = list(tile_compute)
    b = [c + 2 * bT * rad for c in C]
    pc = math.prod(C)
    r_read = math.prod(b) / pc * (h + 2 * bT * rad) / h
    r_comp = sum(math.prod(bi - 2 * T * rad for bi in b) / pc * (h + 2 * rad * (bT - T)) / h
                 for T in range(1, bT + 1)) / bT
    r_read_k = math.prod(tile_loaded) / pc * (h + 2 * bT * rad) / h
    comp = fp_peak * eff / (F * r_comp)
    mem = hbm_gbs * 1e9 * bT / (dtype_bytes * (r_read + 1.0))
    ideal_comp = fp_peak * eff / F
    ideal_mem = hbm_gbs * 1e9 * bT / (2.0 * dtype_bytes)
    return {
        "roof_cells_s": min(comp, mem), "bound": "alu" if comp < mem else "hbm",
        "comp_cells_s": comp, "hbm_cells_s": mem, "R_read": r_read, "R_comp": r_comp,
        "R_read_kernel": r_read_k, "R_comp_kernel": r_read_k,
        "ideal_cells_s": min(ideal_comp, ideal_mem), "flops_per_cell": F, "eff_alu": eff,
        "alg_bytes_per_cell_step": dtype_bytes * (r_read + 1.0) / bT,
        "alg_flops_per_cell_step": F * r_comp,
    }
