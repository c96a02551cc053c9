"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` / ``--impl reference``
legs may import this package.  The product package ``paper_2001_01473_b200`` never imports it and
shares no code with it (the only shared module is ``inputs``, which holds no stencil arithmetic).

Contents
  * :func:`run` -- the plain double-buffered time loop of PAPER.md fig:jacobi2d with
    Table 2's stencil definitions, in C (oracle.c, OpenMP over the outer dimension),
    fp32 or fp64 arithmetic as the run.
  * :func:`run_gradient` -- the same loop for the non-linear gradient2d row of Table 2.
  * :func:`run_system` -- the same loop for a system of n_f arrays updated together, every
    statement reading the previous step of all arrays (NEXT N4).
  * :mod:`oracle.geometry` -- the paper's blocking bookkeeping formulas
    written out independently of the library's C++ (bit-exact checks of an5d_describe /
    an5d_schedule).
(The paper's section-5 performance model lives in the library, an5d_model_paper, and is pinned
directly to Table 5's printed "Model" column by tests/test_model_paper.py.)

Pins (tests/test_oracle_pins.py) tie this oracle to values fixed by the paper and mathematics:
constant field, linear field, quadratic closed form, mirrored impulse, T-fold self-convolution,
brute force on tiny grids.  See DESIGN.md "Oracle and pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2 -ffp-contract=off -fopenmp): IEEE mul/add, no FMA contraction."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
                               "-shared", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB)
        for name, ct in (("oracle_run_f32", ctypes.c_float), ("oracle_run_f64", ctypes.c_double)):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                           ctypes.c_double, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_int64, ctypes.c_int]
        for name in ("oracle_system_f32", "oracle_system_f64"):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                           ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                           ctypes.c_int]
        for name in ("oracle_grad_f32", "oracle_grad_f64"):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return _load().oracle_max_threads()


def run(grid: np.ndarray, rad: int, shape: int, coeffs, divisor: float, T: int, dtype=np.float32,
        nthreads: int = 0) -> np.ndarray:
    """T steps of the naive double-buffered loop on a dense grid (ring included); returns a new array.

    ``coeffs`` is the dense (2r+1)^ndim table (index order outer..x; entry d multiplies the
    neighbour at offset +d), rounded once to ``dtype``; ``divisor`` divides the sum (IEEE division)
    when != 1.  ``nthreads`` <= 0 uses all OpenMP threads.  shape 2 = gradient2d: see
    :func:`run_gradient` (c = the table's centre, c_0 = ``divisor``).
    """
    if shape == 2:   # gradient2d (Table 2): centre entry of the 3x3 table, c_0 = divisor
        c = np.asarray(coeffs, dtype=np.float64).reshape(3, 3)
        return run_gradient(grid, float(c[1, 1]), float(divisor), T, dtype, nthreads)
    lib = _load()
    g = np.ascontiguousarray(grid, dtype=dtype)
    out = np.empty_like(g)
    ext = (ctypes.c_int64 * g.ndim)(*g.shape)
    c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64).reshape(-1))
    fn = lib.oracle_run_f32 if g.dtype == np.float32 else lib.oracle_run_f64
    nt = nthreads if nthreads > 0 else lib.oracle_max_threads()
    rc = fn(g.ndim, int(rad), int(shape), c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(divisor), ext,
            g.ctypes.data, out.ctypes.data, int(T), int(nt))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return out


def run_gradient(grid: np.ndarray, centre: float, c0: float, T: int, dtype=np.float32,
                 nthreads: int = 0) -> np.ndarray:
    """T steps of gradient2d (Table 2) on a dense 2D grid (ring of width 1
    included), in ``dtype``: f' = c f + 1 / sqrt(c_0 + sum_{i=-1,+1} ((f - f_{x+i})^2 + (f - f_{y+i})^2)).
    ``centre`` = c, ``c0`` = c_0, both rounded once to ``dtype``."""
    lib = _load()
    g = np.ascontiguousarray(grid, dtype=dtype)
    if g.ndim != 2:
        raise ValueError("gradient2d is 2D")
    out = np.empty_like(g)
    ext = (ctypes.c_int64 * 2)(*g.shape)
    fn = lib.oracle_grad_f32 if g.dtype == np.float32 else lib.oracle_grad_f64
    nt = nthreads if nthreads > 0 else lib.oracle_max_threads()
    rc = fn(float(centre), float(c0), ext, g.ctypes.data, out.ctypes.data, int(T), int(nt))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return out


def run_system(fields: np.ndarray, rad: int, shape: int, coeffs, T: int, dtype=np.float32,
               nthreads: int = 0) -> np.ndarray:
    """T steps of a multi-field system (NEXT N4) on ``fields`` of shape (n_f, *grid) (rings
    included): A_i' = sum_j sum_d c[i, j][d] A_j[x + d] over the Table-2 taps of ``shape``.
    ``coeffs``: shape (n_f, n_f, (2r+1,)*ndim); block [i, j] is field j's contribution to field i,
    rounded once to ``dtype``.  Returns a new (n_f, *grid) array."""
    lib = _load()
    f = np.ascontiguousarray(fields, dtype=dtype)
    nf = f.shape[0]
    grid = f.shape[1:]
    c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64))
    if c.shape[:2] != (nf, nf):
        raise ValueError("coeffs must be (n_f, n_f, table)")
    c = c.reshape(-1)
    out = np.empty_like(f)
    ext = (ctypes.c_int64 * len(grid))(*grid)
    fn = lib.oracle_system_f32 if f.dtype == np.float32 else lib.oracle_system_f64
    nt = nthreads if nthreads > 0 else lib.oracle_max_threads()
    rc = fn(len(grid), int(rad), int(shape), int(nf), c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ext,
            f.ctypes.data, out.ctypes.data, int(T), int(nt))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return out
