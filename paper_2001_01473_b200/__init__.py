"""paper_2001_01473_b200 -- B200-native N.5D temporally blocked stencils (AN5D, arXiv 2001.01473).

Thin Python binding over the C ABI in ``include/an5d.h`` (libAN5D.so, sm_100a).  Argument
marshalling only: every step of the sweep runs in the library's CUDA kernels.  PyTorch provides
device memory and streams.  There is no CPU fallback: libAN5D.so is loaded on first use (the first
Stencil, schedule() or version() call, or load()), and that call raises ImportError if the library
is missing or fails to load.  Loading lazily keeps the pure-Python host modules of this package
(slab partitioning, perf accounting) importable on a CPU box without the library.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AN5D_LIB") or os.path.join(_HERE, "libAN5D.so")

STAR, BOX, GRAD = 0, 1, 2   # GRAD: gradient2d (Table 2)
F32, F64 = 0, 1

STATUS = {
    0: "AN5D_OK", 1: "AN5D_ERR_INVALID_ARGUMENT", 2: "AN5D_ERR_INFEASIBLE_CONFIG",
    3: "AN5D_ERR_BLOCK_TOO_LARGE", 4: "AN5D_ERR_SHAPE_MISMATCH", 5: "AN5D_ERR_UNSUPPORTED",
    6: "AN5D_ERR_CUDA", 7: "AN5D_ERR_OUT_OF_MEMORY", 8: "AN5D_ERR_NCCL",
}


class AN5DError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("bT", ctypes.c_int), ("bS", ctypes.c_int * 2), ("h", ctypes.c_int64), ("vec", ctypes.c_int),
                ("direct", ctypes.c_int), ("n_thr", ctypes.c_int)]

    def as_dict(self):
        return {"bT": self.bT, "bS": list(self.bS), "h": self.h, "vec": self.vec, "direct": self.direct,
                "n_thr": self.n_thr}


class Geometry(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int), ("rad", ctypes.c_int), ("bT", ctypes.c_int),
        ("interior", ctypes.c_int64 * 3), ("bS", ctypes.c_int * 2), ("bS_loaded", ctypes.c_int * 2),
        ("compute", ctypes.c_int * 2), ("halo_loaded", ctypes.c_int * 2), ("n_tiles", ctypes.c_int64 * 2),
        ("n_tb", ctypes.c_int64), ("h", ctypes.c_int64), ("n_stream_blocks", ctypes.c_int64),
        ("n_tb_prime", ctypes.c_int64), ("stream_overlap", ctypes.c_int64), ("n_thr", ctypes.c_int),
        ("units_per_block", ctypes.c_int), ("grid_blocks", ctypes.c_int64), ("smem_bytes", ctypes.c_size_t),
        ("regs_per_thread", ctypes.c_int), ("vec", ctypes.c_int), ("n_units", ctypes.c_int64),
    ]

    def as_dict(self):
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = list(v) if hasattr(v, "__len__") else v
        return out


class PeerStore(ctypes.Structure):
    _fields_ = [("peer_dst", ctypes.c_void_p * 2), ("peer_plane_shift", ctypes.c_int64 * 2),
                ("send_planes", ctypes.c_int64 * 2)]


class SlabLinks(ctypes.Structure):
    _fields_ = [("peer_bufs", (ctypes.c_void_p * 2) * 2), ("peer_plane_shift", ctypes.c_int64 * 2),
                ("peer_flag", ctypes.c_void_p * 2), ("flag", ctypes.c_void_p), ("epoch", ctypes.c_uint32)]


class DeviceParams(ctypes.Structure):
    _fields_ = [("n_sm", ctypes.c_int), ("max_threads_per_sm", ctypes.c_int), ("peak_comp_gflops", ctypes.c_double),
                ("peak_gm_gbs", ctypes.c_double), ("peak_sm_gbs", ctypes.c_double)]


class ModelResult(ctypes.Structure):
    _fields_ = [("th_comp", ctypes.c_double), ("th_sm_read", ctypes.c_double), ("th_sm_write", ctypes.c_double),
                ("th_gm_read", ctypes.c_double), ("th_gm_write", ctypes.c_double), ("n_tb", ctypes.c_int64),
                ("n_tb_prime", ctypes.c_int64), ("n_thr", ctypes.c_int), ("flops_per_cell", ctypes.c_double),
                ("eff_alu", ctypes.c_double), ("eff_sm", ctypes.c_double), ("time_comp", ctypes.c_double),
                ("time_sm", ctypes.c_double), ("time_gm", ctypes.c_double), ("time_model", ctypes.c_double),
                ("gflops", ctypes.c_double), ("bottleneck", ctypes.c_int)]

    def as_dict(self):
        d = {name: getattr(self, name) for name, _ in self._fields_}
        d["bottleneck"] = ("comp", "sm", "gm")[self.bottleneck]
        return d


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libAN5D.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    pi64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "an5d_create": (I32, [I32, I32, I32, ctypes.POINTER(ctypes.c_double), ctypes.c_size_t, D, I32,
                              ctypes.POINTER(P)]),
        "an5d_run": (I32, [P, P, P, pi64, pi64, I64, ctypes.POINTER(Config), P]),
        "an5d_sweep": (I32, [P, P, P, pi64, pi64, I32, ctypes.POINTER(Config), I64, I64, I64, I64, P, P]),
        "an5d_copy_ring": (I32, [P, P, P, pi64, pi64, I64, I64, P]),
        "an5d_sweep_peer": (I32, [P, P, P, pi64, pi64, I32, ctypes.POINTER(Config), I64, I64, I64, I64,
                                  ctypes.POINTER(PeerStore), P, P]),
        "an5d_run_slab": (I32, [P, P, P, pi64, pi64, I64, ctypes.POINTER(Config), I64, I64, I64, I64,
                                ctypes.POINTER(SlabLinks), P]),
        "an5d_stream_signal": (I32, [P, ctypes.c_uint32, P]),
        "an5d_stream_wait": (I32, [P, ctypes.c_uint32, P]),
        "an5d_ipc_export": (I32, [P, P, pi64]),
        "an5d_ipc_open": (I32, [P, ctypes.POINTER(P)]),
        "an5d_ipc_close": (I32, [P]),
        "an5d_plan_config": (I32, [P, pi64, I64, ctypes.POINTER(Config), ctypes.POINTER(Config)]),
        "an5d_describe": (I32, [P, pi64, ctypes.POINTER(Config), ctypes.POINTER(Geometry)]),
        "an5d_tune": (I32, [P, P, P, pi64, pi64, I64, ctypes.POINTER(Config), I32, ctypes.POINTER(Config),
                            ctypes.POINTER(ctypes.c_double), P]),
        "an5d_schedule": (I32, [I64, I32, ctypes.POINTER(ctypes.c_int), I64, pi64, ctypes.POINTER(ctypes.c_int)]),
        "an5d_model_paper": (I32, [I32, I32, I32, I32, I32, pi64, I32, ctypes.POINTER(ctypes.c_int), I64,
                                   ctypes.POINTER(DeviceParams), ctypes.POINTER(ModelResult)]),
        "an5d_model_paper_search": (I32, [I32, I32, I32, I32, I32, pi64, ctypes.POINTER(DeviceParams), I32,
                                          ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_int)]),
        "an5d_create_system": (I32, [I32, I32, I32, I32, ctypes.POINTER(ctypes.c_double), ctypes.c_size_t, I32,
                                     ctypes.POINTER(P)]),
        "an5d_comm_unique_id": (I32, [P]),
        "an5d_set_comm": (I32, [P, P, I32, I32, I64, I64, I32]),
        "an5d_last_launch_count": (I64, [P]),
        "an5d_destroy": (I32, [P]),
        "an5d_last_error": (ctypes.c_char_p, []),
        "an5d_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _LazyLib:
    """Loads libAN5D.so on first attribute access (raises ImportError if it is missing)."""

    _h = None

    def __getattr__(self, name):
        if _LazyLib._h is None:
            _LazyLib._h = _load()
        return getattr(_LazyLib._h, name)


_lib = _LazyLib()


def load():
    """Load libAN5D.so now (raises ImportError if it is missing or does not load); returns the CDLL."""
    _lib.an5d_version
    return _LazyLib._h


def loaded() -> bool:
    return _LazyLib._h is not None

EXPORTED_SYMBOLS = ("an5d_create", "an5d_create_system", "an5d_comm_unique_id", "an5d_set_comm", "an5d_run", "an5d_sweep", "an5d_sweep_peer", "an5d_run_slab", "an5d_stream_signal",
                    "an5d_stream_wait", "an5d_ipc_export", "an5d_ipc_open", "an5d_ipc_close", "an5d_copy_ring", "an5d_plan_config", "an5d_tune",
                    "an5d_describe", "an5d_schedule", "an5d_model_paper", "an5d_model_paper_search",
                    "an5d_last_launch_count", "an5d_destroy", "an5d_last_error", "an5d_version")


def _check(st: int):
    if st != 0:
        raise AN5DError(st, _lib.an5d_last_error().decode())


def _i64(vals):
    arr = (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])
    return arr


def _cfg(cfg) -> Config | None:
    if cfg is None:
        return None
    if isinstance(cfg, Config):
        return cfg
    c = Config()
    c.bT = int(cfg.get("bT", 0))
    bs = cfg.get("bS", (0, 0)) or (0, 0)
    c.bS[0] = int(bs[0]) if len(bs) > 0 else 0
    c.bS[1] = int(bs[1]) if len(bs) > 1 else 0
    c.h = int(cfg.get("h", 0))
    c.vec = int(cfg.get("vec", 0))
    c.direct = int(cfg.get("direct", 0))
    c.n_thr = int(cfg.get("n_thr", 0) or 0)
    return c


def schedule(T: int, bT: int):
    """Sweep degrees of the host loop (reading R-7) and trailing-copy flag."""
    n = ctypes.c_int64()
    tc = ctypes.c_int()
    _check(_lib.an5d_schedule(int(T), int(bT), None, 0, ctypes.byref(n), ctypes.byref(tc)))
    buf = (ctypes.c_int * max(1, n.value))()
    _check(_lib.an5d_schedule(int(T), int(bT), buf, n.value, ctypes.byref(n), ctypes.byref(tc)))
    return [buf[i] for i in range(n.value)], bool(tc.value)


def _devparams(dev: dict) -> DeviceParams:
    d = DeviceParams()
    d.n_sm = int(dev["n_sm"])
    d.max_threads_per_sm = int(dev.get("max_threads_per_sm", 2048))
    d.peak_comp_gflops = float(dev["comp"])
    d.peak_gm_gbs = float(dev["gm"])
    d.peak_sm_gbs = float(dev["sm"])
    return d


def model_paper(ndim, rad, shape, has_div, dtype, interior, bT, bS, h, dev) -> dict:
    """The paper's section-5 model (an5d_model_paper) for one configuration.
    dev: {"n_sm", "comp" (GFLOP/s of the dtype), "gm" (GB/s), "sm" (GB/s)} (Table 4)."""
    out = ModelResult()
    bs = (ctypes.c_int * 2)(*(list(bS) + [0, 0])[:2])
    dt = F32 if dtype in (torch.float32, F32) else F64
    _check(_lib.an5d_model_paper(ndim, rad, shape, int(bool(has_div)), dt, _i64(interior), int(bT), bs, int(h),
                                 ctypes.byref(_devparams(dev)), ctypes.byref(out)))
    return out.as_dict()


def model_paper_search(ndim, rad, shape, has_div, dtype, interior, dev, top_k=5):
    """The paper's "Tuned" search space ranked by the model (an5d_model_paper_search):
    returns (list of (config dict, GFLOP/s) best first, number of feasible configurations)."""
    cfgs = (Config * max(1, top_k))()
    gf = (ctypes.c_double * max(1, top_k))()
    n = ctypes.c_int()
    dt = F32 if dtype in (torch.float32, F32) else F64
    _check(_lib.an5d_model_paper_search(ndim, rad, shape, int(bool(has_div)), dt, _i64(interior),
                                        ctypes.byref(_devparams(dev)), int(top_k), cfgs, gf, ctypes.byref(n)))
    return [(cfgs[i].as_dict(), gf[i]) for i in range(min(top_k, n.value))], n.value


def vec_width(dtype) -> int:
    return 4 if dtype in (torch.float32, F32) else 2


def empty_grid(extents, rad: int, dtype=torch.float32, device="cuda"):
    """Allocate a grid view meeting the vector-path alignment contract of an5d.h.

    Rows are padded to a multiple of 128 bytes and the view starts so that element x = rad (the
    first interior cell of every row) is 16-byte aligned.
    """
    extents = [int(e) for e in extents]
    elem = torch.empty((), dtype=dtype).element_size()
    A = 16 // elem
    pitch = -(-extents[-1] // (128 // elem)) * (128 // elem)
    strides = [1]
    if len(extents) >= 2:
        strides.insert(0, pitch)
    if len(extents) == 3:
        strides.insert(0, pitch * extents[1])
    n = strides[0] * extents[0] + 2 * A
    buf = torch.empty(n, dtype=dtype, device=device)
    off = (A - rad % A) % A
    return torch.as_strided(buf, extents, strides, storage_offset=off)


def to_grid(t: torch.Tensor, rad: int):
    """Copy a tensor into an aligned grid view (see empty_grid)."""
    g = empty_grid(t.shape, rad, t.dtype, t.device)
    g.copy_(t)
    return g


def _geom_of(t: torch.Tensor):
    if not t.is_cuda:
        raise ValueError("grids must be CUDA tensors (no CPU path)")
    if t.dtype not in (torch.float32, torch.float64):
        raise ValueError("grid dtype must be float32 or float64")
    if t.dim() not in (2, 3) or t.stride(-1) != 1:
        raise ValueError("grid must be 2D/3D with unit x stride")
    return list(t.shape), [t.stride(i) for i in range(t.dim() - 1)]


class Stencil:
    """One stencil (an5d_create): ndim 2|3, radius 1..4, STAR|BOX, dense coefficient table.

    ``coeffs``: array-like of shape (2r+1,)*ndim, index order (d_outer..d_x); entry d multiplies
    the neighbour at offset +d.  ``divisor``: j-stencil c_0 (Table 2), 1.0 for none.
    """

    def __init__(self, ndim: int, rad: int, shape: int, coeffs, divisor: float = 1.0, dtype=torch.float32):
        import numpy as np

        c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64).reshape(-1))
        self.ndim, self.rad, self.shape, self.divisor = ndim, rad, shape, float(divisor)
        self.dtype = dtype
        self.coeffs = c
        dt = F32 if dtype == torch.float32 else F64
        h = ctypes.c_void_p()
        _check(_lib.an5d_create(ndim, rad, shape, c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                c.size, float(divisor), dt, ctypes.byref(h)))
        self._h = h

    @staticmethod
    def _geom(t: torch.Tensor):
        return _geom_of(t)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.an5d_destroy(h)
            self._h = None

    # -- run / sweep ---------------------------------------------------------------------------
    def run(self, grid_in: torch.Tensor, grid_out: torch.Tensor, T: int, cfg=None, stream=None):
        """Advance T steps; result in grid_out (grid_in's interior is clobbered for T >= 2)."""
        ext, pit = self._geom(grid_in)
        if list(grid_out.shape) != list(grid_in.shape) or grid_out.stride() != grid_in.stride():
            raise ValueError("grid_in and grid_out must have identical shape and strides")
        if grid_in.dtype != self.dtype or grid_out.dtype != self.dtype:
            raise ValueError("grid dtype does not match the stencil dtype")
        st = stream if stream is not None else torch.cuda.current_stream(grid_in.device)
        c = _cfg(cfg)
        _check(_lib.an5d_run(self._h, grid_in.data_ptr(), grid_out.data_ptr(), _i64(ext), _i64(pit), int(T),
                             ctypes.byref(c) if c is not None else None, ctypes.c_void_p(st.cuda_stream)))
        return grid_out

    def sweep(self, src: torch.Tensor, dst: torch.Tensor, degree: int, cfg, outer_offset: int = 0,
              global_outer_extent: int | None = None, out_lo: int | None = None, out_hi: int | None = None,
              write_count: torch.Tensor | None = None, stream=None, peers=None):
        """One sweep of `degree` time steps (slab mode; see an5d.h an5d_sweep).  ``peers``: None or
        a dict {"lo"/"hi": (device pointer int, plane shift, planes)} for the fused halo exchange
        (an5d_sweep_peer)."""
        ext, pit = self._geom(src)
        g = ext[0] if global_outer_extent is None else global_outer_extent
        lo = self.rad if out_lo is None else out_lo
        hi = ext[0] - self.rad if out_hi is None else out_hi
        st = stream if stream is not None else torch.cuda.current_stream(src.device)
        c = _cfg(cfg)
        wc = write_count.data_ptr() if write_count is not None else None
        if peers:
            ps = PeerStore()
            for k, side in enumerate(("lo", "hi")):
                if side in peers and peers[side]:
                    ptr, shift, n = peers[side]
                    ps.peer_dst[k] = int(ptr)
                    ps.peer_plane_shift[k] = int(shift)
                    ps.send_planes[k] = int(n)
            _check(_lib.an5d_sweep_peer(self._h, src.data_ptr(), dst.data_ptr(), _i64(ext), _i64(pit), int(degree),
                                        ctypes.byref(c), int(outer_offset), int(g), int(lo), int(hi), ctypes.byref(ps),
                                        wc, ctypes.c_void_p(st.cuda_stream)))
            return
        _check(_lib.an5d_sweep(self._h, src.data_ptr(), dst.data_ptr(), _i64(ext), _i64(pit), int(degree),
                               ctypes.byref(c), int(outer_offset), int(g), int(lo), int(hi), wc,
                               ctypes.c_void_p(st.cuda_stream)))

    def run_slab(self, grid_in: torch.Tensor, grid_out: torch.Tensor, T: int, cfg, outer_offset: int,
                 global_outer_extent: int, own_lo: int, own_hi: int, lo=None, hi=None, flag: int = 0, epoch: int = 0,
                 stream=None) -> int:
        """One slab's T-step run with the fused halo exchange (an5d_run_slab).  ``lo`` / ``hi``:
        None or (neighbour buffer paired with grid_in, with grid_out, plane shift, flag pointer).
        Returns the new epoch."""
        ext, pit = self._geom(grid_in)
        st = stream if stream is not None else torch.cuda.current_stream(grid_in.device)
        L = SlabLinks()
        for k, side in enumerate((lo, hi)):
            if side:
                b_in, b_out, shift, fl = side
                L.peer_bufs[k][0] = int(b_in)
                L.peer_bufs[k][1] = int(b_out)
                L.peer_plane_shift[k] = int(shift)
                L.peer_flag[k] = int(fl)
        L.flag = int(flag)
        L.epoch = int(epoch)
        c = _cfg(cfg)
        _check(_lib.an5d_run_slab(self._h, grid_in.data_ptr(), grid_out.data_ptr(), _i64(ext), _i64(pit), int(T),
                                  ctypes.byref(c), int(outer_offset), int(global_outer_extent), int(own_lo),
                                  int(own_hi), ctypes.byref(L), ctypes.c_void_p(st.cuda_stream)))
        return int(L.epoch)

    def set_comm(self, unique_id: bytes | None, rank: int = 0, nranks: int = 1, global_outer_extent: int = 0,
                 outer_offset: int = 0, ghost_planes: int = 0):
        """Join an NCCL communicator (an5d_set_comm): later runs treat the grids as this rank's slab
        and exchange ghost planes with ncclSend/ncclRecv inside the library.  None detaches."""
        uid = ctypes.create_string_buffer(unique_id, 128) if unique_id is not None else None
        _check(_lib.an5d_set_comm(self._h, uid, int(rank), int(nranks), int(global_outer_extent), int(outer_offset),
                                  int(ghost_planes)))

    def copy_ring(self, src: torch.Tensor, dst: torch.Tensor, outer_offset: int = 0,
                  global_outer_extent: int | None = None, stream=None):
        ext, pit = self._geom(src)
        g = ext[0] if global_outer_extent is None else global_outer_extent
        st = stream if stream is not None else torch.cuda.current_stream(src.device)
        _check(_lib.an5d_copy_ring(self._h, src.data_ptr(), dst.data_ptr(), _i64(ext), _i64(pit),
                                   int(outer_offset), int(g), ctypes.c_void_p(st.cuda_stream)))

    # -- planner / bookkeeping -------------------------------------------------------------------
    def plan_config(self, extents, T: int = 0, hint=None) -> dict:
        out = Config()
        h = _cfg(hint)
        _check(_lib.an5d_plan_config(self._h, _i64(extents), int(T), ctypes.byref(h) if h else None,
                                     ctypes.byref(out)))
        return out.as_dict()

    def tune(self, grid_in: torch.Tensor, grid_out: torch.Tensor, T: int = 0, hint=None, top_k: int = 5,
             stream=None) -> dict:
        """Model top-k + measured pick (an5d_tune).  Reads grid_in, overwrites grid_out's
        interior; blocks until the candidate sweeps are timed.  Returns the config with the measured
        "seconds_per_cell_step" of the winner."""
        ext, pit = self._geom(grid_in)
        st = stream if stream is not None else torch.cuda.current_stream(grid_in.device)
        out = Config()
        best = ctypes.c_double()
        h = _cfg(hint)
        _check(_lib.an5d_tune(self._h, grid_in.data_ptr(), grid_out.data_ptr(), _i64(ext), _i64(pit), int(T),
                              ctypes.byref(h) if h else None, int(top_k), ctypes.byref(out), ctypes.byref(best),
                              ctypes.c_void_p(st.cuda_stream)))
        d = out.as_dict()
        d["seconds_per_cell_step"] = best.value
        return d

    def describe(self, extents, cfg) -> dict:
        out = Geometry()
        c = _cfg(cfg)
        _check(_lib.an5d_describe(self._h, _i64(extents), ctypes.byref(c), ctypes.byref(out)))
        return out.as_dict()

    def last_launch_count(self) -> int:
        return int(_lib.an5d_last_launch_count(self._h))


def stream_signal(flag_ptr: int, value: int, stream=None):
    """Stream-ordered write of a 32-bit device flag after the stream's prior work (an5d.h)."""
    st = stream if stream is not None else torch.cuda.current_stream()
    _check(_lib.an5d_stream_signal(ctypes.c_void_p(int(flag_ptr)), int(value), ctypes.c_void_p(st.cuda_stream)))


def stream_wait(flag_ptr: int, value: int, stream=None):
    """The stream waits until the 32-bit device flag is >= value (an5d.h)."""
    st = stream if stream is not None else torch.cuda.current_stream()
    _check(_lib.an5d_stream_wait(ctypes.c_void_p(int(flag_ptr)), int(value), ctypes.c_void_p(st.cuda_stream)))


def ipc_export(ptr: int):
    """(64-byte handle, byte offset) of the allocation holding a device pointer (CUDA IPC)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _check(_lib.an5d_ipc_export(ctypes.c_void_p(int(ptr)), h, ctypes.byref(off)))
    return h.raw, off.value


def ipc_open(handle: bytes) -> int:
    """Map another process's allocation (CUDA IPC); returns its base device pointer here."""
    base = ctypes.c_void_p()
    _check(_lib.an5d_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(base)))
    return int(base.value)


def ipc_close(base: int):
    _check(_lib.an5d_ipc_close(ctypes.c_void_p(int(base))))


def comm_unique_id() -> bytes:
    """128-byte NCCL unique id for an5d_set_comm (call on rank 0, broadcast to the others)."""
    b = ctypes.create_string_buffer(128)
    _check(_lib.an5d_comm_unique_id(b))
    return b.raw


def version() -> str:
    return _lib.an5d_version().decode()


def empty_fields(n_fields: int, extents, rad: int, dtype=torch.float32, device="cuda"):
    """n_fields grids of identical layout (see empty_grid), field-major in one allocation: a view of
    shape (n_fields, *extents) whose field stride is a multiple of 128 bytes (an5d_create_system)."""
    extents = [int(e) for e in extents]
    elem = torch.empty((), dtype=dtype).element_size()
    A = 16 // elem
    pitch = -(-extents[-1] // (128 // elem)) * (128 // elem)
    strides = [1]
    if len(extents) >= 2:
        strides.insert(0, pitch)
    if len(extents) == 3:
        strides.insert(0, pitch * extents[1])
    fstride = -(-(strides[0] * extents[0]) // (128 // elem)) * (128 // elem)
    buf = torch.empty(fstride * n_fields + 2 * A, dtype=dtype, device=device)
    off = (A - rad % A) % A
    return torch.as_strided(buf, [n_fields] + extents, [fstride] + strides, storage_offset=off)


def to_fields(t: torch.Tensor, rad: int):
    """Copy a (n_fields, *grid) tensor into an aligned field-major view (see empty_fields)."""
    g = empty_fields(t.shape[0], t.shape[1:], rad, t.dtype, t.device)
    g.copy_(t)
    return g


class System(Stencil):
    """A multi-field system (an5d_create_system; NEXT N4): n_fields arrays advance together,
    statement i reading the previous step of every array through block [i, j] of ``coeffs``
    (shape (n_fields, n_fields, (2r+1,)*ndim)).  Grids are (n_fields, *extents) tensors from
    empty_fields / to_fields; run / sweep / tune / copy_ring / describe as for Stencil."""

    def __init__(self, ndim: int, rad: int, shape: int, coeffs, dtype=torch.float32):
        import numpy as np

        c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64))
        nf = c.shape[0]
        if c.shape[:2] != (nf, nf):
            raise ValueError("coeffs must have shape (n_fields, n_fields, table)")
        c = c.reshape(-1)
        self.ndim, self.rad, self.shape, self.divisor, self.n_fields = ndim, rad, shape, 1.0, nf
        self.dtype = dtype
        self.coeffs = c
        dt = F32 if dtype == torch.float32 else F64
        h = ctypes.c_void_p()
        _check(_lib.an5d_create_system(ndim, rad, shape, nf, c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                       c.size, dt, ctypes.byref(h)))
        self._h = h

    @staticmethod
    def _geom(t: torch.Tensor):
        """(n_fields, *grid) tensor -> extents of one grid, pitches = [field stride, grid pitches]."""
        if not t.is_cuda:
            raise ValueError("grids must be CUDA tensors (no CPU path)")
        if t.dtype not in (torch.float32, torch.float64) or t.dim() not in (3, 4) or t.stride(-1) != 1:
            raise ValueError("fields must be a (n_fields, *grid) float32/float64 tensor with unit x stride")
        return list(t.shape[1:]), [t.stride(i) for i in range(t.dim() - 1)]
