"""Slab decomposition of the streaming dimension across GPUs (BASELINE north_star (d)).

The paper is single-GPU; its "division of the streaming dimension" into stream blocks
is the geometry reused here: rank k owns a contiguous run of interior planes of the OUTERMOST
(streaming) dimension and holds G = b_T * rad ghost planes on each side that has a neighbour.
Every sweep of degree d:

  1. the BOUNDARY output planes (the lowest / highest owned planes a neighbour needs next sweep)
     are computed first, on the caller's stream;
  2. their outermost d_next * rad planes are exchanged with rank-1 / rank+1 (send owned planes,
     receive into ghost planes of the same destination buffer) on a separate comm stream;
  3. the INTERIOR output planes are computed on the caller's stream while the exchange runs;
  4. the next sweep waits for both.

Bookkeeping (:class:`SlabPlan`) is pure integer host logic, shared by the NCCL runner
(:func:`run_distributed`, one process per GPU), the in-process loopback runner used for single-GPU
tests (:func:`run_loopback`) and the world-size-2 gloo CPU tests.  The compute itself is the
library's ``an5d_sweep`` in slab mode (outer_offset / global_outer_extent, include/an5d.h); the
exchange is torch.distributed send/recv (NCCL over NVLink on the GPU box).
"""
from __future__ import annotations

import dataclasses
import json
import os
import statistics
import time


@dataclasses.dataclass(frozen=True)
class Slab:
    rank: int
    nranks: int
    gE0: int          # global outermost extent (ring planes included)
    rad: int
    G: int            # ghost depth (planes) = b_T * rad
    own_lo: int       # owned global interior planes [own_lo, own_hi)
    own_hi: int
    loc_lo: int       # global planes held locally [loc_lo, loc_hi) (owned + ghosts / global ring)
    loc_hi: int

    @property
    def n_local(self) -> int:
        return self.loc_hi - self.loc_lo

    @property
    def out_lo(self) -> int:      # owned planes in local coordinates
        return self.own_lo - self.loc_lo

    @property
    def out_hi(self) -> int:
        return self.own_hi - self.loc_lo

    @property
    def has_lower(self) -> bool:
        return self.rank > 0

    @property
    def has_upper(self) -> bool:
        return self.rank < self.nranks - 1


def partition(gE0: int, rad: int, nranks: int, G: int, align: int = 1):
    """Contiguous owned chunks of the global interior planes [rad, gE0 - rad).

    chunk = ceil(I / n) rounded up to a multiple of ``align`` (the stream-block length, so slabs
    add no redundancy beyond the single-GPU stream overlap); every rank must own at
    least G planes (a ghost region never spans two ranks).
    """
    I = gE0 - 2 * rad
    if nranks < 1 or I < nranks:
        raise ValueError(f"cannot split {I} interior planes over {nranks} ranks")
    chunk = -(-I // nranks)
    chunk = -(-chunk // align) * align
    out = []
    for k in range(nranks):
        lo = rad + min(I, k * chunk)
        hi = rad + min(I, (k + 1) * chunk)
        if hi - lo < G and nranks > 1:
            raise ValueError(f"rank {k} owns {hi - lo} planes < ghost depth {G}; use fewer ranks")
        out.append(Slab(k, nranks, gE0, rad, G, lo, hi, max(0, lo - G), min(gE0, hi + G)))
    return out


def partition_aligned(gE0: int, rad: int, nranks: int, G: int, h: int):
    """:func:`partition` with owned chunks a multiple of the stream-block length h (SURVEY.md
    §8(e): slab boundaries then fall on stream-block boundaries, so slabs add no stream-block
    overlap beyond the single-GPU one), falling back to unaligned chunks when aligning would leave
    a rank with fewer than G planes."""
    if h > 1:
        try:
            parts = partition(gE0, rad, nranks, G, align=h)
            if all(p.own_hi - p.own_lo >= max(1, G if nranks > 1 else 1) for p in parts):
                return parts
        except ValueError:
            pass
    return partition(gE0, rad, nranks, G, align=1)


@dataclasses.dataclass(frozen=True)
class SweepParts:
    """Output-plane ranges (local coordinates) of one sweep on one slab."""
    boundary: tuple   # ranges computed before the exchange
    interior: tuple   # ranges computed concurrently with the exchange
    sends: tuple      # (peer, local_lo, n_planes): owned planes sent to peer
    recvs: tuple      # (peer, local_lo, n_planes): ghost planes received from peer


def sweep_parts(s: Slab, next_degree: int, h: int) -> SweepParts:
    """Split the owned planes of a sweep into boundary and interior parts and list the exchange
    for a following sweep of degree ``next_degree`` (0 = none): it needs next_degree * rad ghost
    planes per neighbour side."""
    g = next_degree * s.rad
    lo, hi = s.out_lo, s.out_hi
    hb = max(g, h)
    blo = lo + hb if (s.has_lower and g) else lo          # [lo, blo) boundary below
    bhi = hi - hb if (s.has_upper and g) else hi          # [bhi, hi) boundary above
    if blo >= bhi:                                        # slab too thin to overlap
        boundary, interior = ((lo, hi),), ()
    else:
        boundary = tuple(r for r in ((lo, blo), (bhi, hi)) if r[1] > r[0])
        interior = ((blo, bhi),)
    sends, recvs = [], []
    if g:
        if s.has_lower:
            sends.append((s.rank - 1, lo, g))
            recvs.append((s.rank - 1, lo - g, g))
        if s.has_upper:
            sends.append((s.rank + 1, hi - g, g))
            recvs.append((s.rank + 1, hi, g))
    return SweepParts(boundary, interior, tuple(sends), tuple(recvs))


def local_extents(s: Slab, inner_extents):
    return (s.n_local,) + tuple(int(e) for e in inner_extents)


# ---------------------------------------------------------------------------------------------
# Runners
# ---------------------------------------------------------------------------------------------
def _plane_view(buf, lo, n):
    """Contiguous flat view of local planes [lo, lo + n) of a (possibly padded) grid view."""
    import torch
    pz = buf.stride(0)
    flat = torch.empty(0, dtype=buf.dtype, device=buf.device).set_(buf.untyped_storage())
    start = buf.storage_offset() + lo * pz
    return flat[start:start + n * pz]


def run_distributed(stencil, s: Slab, bufs, T: int, cfg: dict, group=None, comm_stream=None,
                    schedule_fn=None):
    """One rank's share of a T-step run (torch.distributed already initialised; NCCL on GPUs).

    ``bufs`` = (grid_in, grid_out) local slab arrays (ghosts included), grid_in holding the input
    on every local plane.  On return grid_out's owned planes hold step T.  ``stencil`` is a
    :class:`paper_2001_01473_b200.Stencil` (or any object with the same sweep/copy_ring API).
    """
    import torch
    import torch.distributed as dist

    from . import schedule as lib_schedule
    degrees, trailing = (schedule_fn or lib_schedule)(T, cfg["bT"])
    a, b = bufs
    main = torch.cuda.current_stream() if a.is_cuda else None
    comm = comm_stream if comm_stream is not None else (torch.cuda.Stream(a.device) if a.is_cuda else None)
    gE0 = s.gE0
    stencil.copy_ring(a, b, outer_offset=s.loc_lo, global_outer_extent=gE0)
    ev_prev = None
    for i, d in enumerate(degrees):
        src, dst = (a, b) if i % 2 == 0 else (b, a)
        nd = degrees[i + 1] if i + 1 < len(degrees) else 0
        parts = sweep_parts(s, nd, int(cfg.get("h") or 0))
        if ev_prev is not None and main is not None:
            main.wait_event(ev_prev)
        for lo, hi in parts.boundary:
            stencil.sweep(src, dst, d, cfg, outer_offset=s.loc_lo, global_outer_extent=gE0, out_lo=lo, out_hi=hi)
        if parts.sends or parts.recvs:
            if main is not None:
                ev_b = torch.cuda.Event()
                ev_b.record(main)
                with torch.cuda.stream(comm):
                    comm.wait_event(ev_b)
                    _exchange(dst, parts, group)
                    ev_prev = torch.cuda.Event()
                    ev_prev.record(comm)
            else:
                _exchange(dst, parts, group)
        for lo, hi in parts.interior:
            stencil.sweep(src, dst, d, cfg, outer_offset=s.loc_lo, global_outer_extent=gE0, out_lo=lo, out_hi=hi)
    if ev_prev is not None and main is not None:
        main.wait_event(ev_prev)
    if trailing:
        # b_T == 1 with an even sweep count: the result sits in grid_in; copy the owned planes
        n = s.out_hi - s.out_lo
        _plane_view(b, s.out_lo, n).copy_(_plane_view(a, s.out_lo, n))
    return b


def _exchange(dst, parts: SweepParts, group):
    import torch.distributed as dist
    ops = []
    for peer, lo, n in parts.recvs:
        ops.append(dist.P2POp(dist.irecv, _plane_view(dst, lo, n), peer, group))
    for peer, lo, n in parts.sends:
        ops.append(dist.P2POp(dist.isend, _plane_view(dst, lo, n).contiguous(), peer, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def run_loopback(stencil, slabs, bufs_per_slab, T: int, cfg: dict, schedule_fn=None):
    """All slabs in one process on one device, ghost planes exchanged by device copies: the same
    partition, sweep split and slab-mode sweeps as :func:`run_distributed` (single-GPU CI of the
    multi-GPU bookkeeping, SURVEY.md §4 "loopback mode")."""
    from . import schedule as lib_schedule
    degrees, trailing = (schedule_fn or lib_schedule)(T, cfg["bT"])
    for s, (a, b) in zip(slabs, bufs_per_slab):
        stencil.copy_ring(a, b, outer_offset=s.loc_lo, global_outer_extent=s.gE0)
    for i, d in enumerate(degrees):
        nd = degrees[i + 1] if i + 1 < len(degrees) else 0
        plist = []
        for s, (a, b) in zip(slabs, bufs_per_slab):
            src, dst = (a, b) if i % 2 == 0 else (b, a)
            parts = sweep_parts(s, nd, int(cfg.get("h") or 0))
            plist.append((parts, dst))
            for lo, hi in parts.boundary + parts.interior:
                stencil.sweep(src, dst, d, cfg, outer_offset=s.loc_lo, global_outer_extent=s.gE0,
                              out_lo=lo, out_hi=hi)
        for k, (parts, dst) in enumerate(plist):
            for peer, lo, n in parts.recvs:
                ppart, pdst = plist[peer]
                # the peer's matching send: same length, the side facing rank k
                (sl,) = [x for x in ppart.sends if x[0] == k]
                _plane_view(dst, lo, n).copy_(_plane_view(pdst, sl[1], n))
    if trailing:
        for s, (a, b) in zip(slabs, bufs_per_slab):
            n = s.out_hi - s.out_lo
            _plane_view(b, s.out_lo, n).copy_(_plane_view(a, s.out_lo, n))
    return [b for _, b in bufs_per_slab]


# ---------------------------------------------------------------------------------------------
# Fused halo exchange: the boundary planes are stored into the
# neighbours' ghost planes by the sweep kernel itself (an5d_sweep_peer); stream-ordered flags
# order the slabs.  No separate exchange step, no NCCL on the data path.
# ---------------------------------------------------------------------------------------------
@dataclasses.dataclass
class PeerLink:
    """One neighbour as seen from this rank: its two slab buffers (device pointers valid on this
    device, same parity order as ours), its plane shift (our loc_lo - its loc_lo) and its
    progress flag (uint32 device pointer)."""
    bufs: tuple
    shift: int
    flag: int


@dataclasses.dataclass
class FusedLinks:
    lo: PeerLink | None
    hi: PeerLink | None
    flag: int          # this rank's progress flag (uint32 device pointer)
    counter: list = dataclasses.field(default_factory=lambda: [0])   # shared epoch holder

    @property
    def epoch(self) -> int:
        """Sweeps completed by every rank in earlier runs (flags are never reset)."""
        return self.counter[0]

    @epoch.setter
    def epoch(self, v: int):
        self.counter[0] = v

    def swapped(self) -> "FusedLinks":
        """The same links for runs whose (grid_in, grid_out) are this one's (grid_out, grid_in):
        the neighbours' buffers swapped, the SAME flags and epoch (the ordering spans runs)."""
        sw = lambda ln: None if ln is None else PeerLink((ln.bufs[1], ln.bufs[0]), ln.shift, ln.flag)
        return FusedLinks(sw(self.lo), sw(self.hi), self.flag, self.counter)


def run_fused(stencil, s: Slab, bufs, T: int, cfg: dict, links: FusedLinks, stream=None, schedule_fn=None):
    """One rank's share of a T-step run with the fused halo exchange, entirely in the library
    (an5d_run_slab, stream-ordered): before sweep i a rank waits until both neighbours finished
    sweep i-1 (flag >= epoch + i) -- its ghost planes for sweep i are then stored, and the
    neighbours no longer read the buffer sweep i writes ghosts into; sweep i stores the
    d_next * rad outermost owned planes into the neighbours' buffers of its destination's parity
    (from the sweep kernel); then the rank writes flag = epoch + i + 1.  Returns grid_out."""
    a, b = bufs
    side = lambda ln: None if ln is None else (ln.bufs[0], ln.bufs[1], ln.shift, ln.flag)
    links.epoch = stencil.run_slab(a, b, T, cfg, s.loc_lo, s.gE0, s.out_lo, s.out_hi, lo=side(links.lo),
                                   hi=side(links.hi), flag=links.flag, epoch=links.epoch, stream=stream)
    return b


def connect_fused(slabs, rank: int, bufs, flag, group=None):
    """Multi-process setup of the fused exchange (one process per GPU): every rank exports CUDA IPC
    handles of its two slab buffers and its flag, all ranks gather them (torch.distributed), and
    each rank maps its neighbours' (NVLink peer mappings on a multi-GPU box).  Returns
    (FusedLinks, opened bases to close with an5d.ipc_close)."""
    import torch.distributed as dist
    import paper_2001_01473_b200 as an5d
    mine = [an5d.ipc_export(t.data_ptr()) for t in (bufs[0], bufs[1], flag)]
    allh = [None] * len(slabs)
    dist.all_gather_object(allh, mine, group=group)
    s = slabs[rank]
    opened, links = [], {}
    for side, k in (("lo", rank - 1), ("hi", rank + 1)):
        if 0 <= k < len(slabs):
            ptrs = []
            for h, off in allh[k]:
                base = an5d.ipc_open(h)
                opened.append(base)
                ptrs.append(base + off)
            links[side] = PeerLink((ptrs[0], ptrs[1]), s.loc_lo - slabs[k].loc_lo, ptrs[2])
    return FusedLinks(links.get("lo"), links.get("hi"), flag.data_ptr()), opened


def loopback_fused(stencil, slabs, bufs_per_slab, T: int, cfg: dict, schedule_fn=None):
    """All slabs on ONE device, one CUDA stream per slab, peer pointers = the other slabs'
    buffers: the fused exchange's kernel-side peer stores and its flag protocol, with the slabs
    genuinely running concurrently (single-GPU test of the multi-GPU data path)."""
    import torch
    dev = bufs_per_slab[0][0].device
    n = len(slabs)
    flags = torch.zeros(n * 32, dtype=torch.int32, device=dev)   # one flag per 128-byte line
    fptr = lambda k: flags.data_ptr() + 128 * k
    links = []
    for k, s in enumerate(slabs):
        lo = PeerLink(tuple(t.data_ptr() for t in bufs_per_slab[k - 1]), s.loc_lo - slabs[k - 1].loc_lo,
                      fptr(k - 1)) if k > 0 else None
        hi = PeerLink(tuple(t.data_ptr() for t in bufs_per_slab[k + 1]), s.loc_lo - slabs[k + 1].loc_lo,
                      fptr(k + 1)) if k + 1 < n else None
        links.append(FusedLinks(lo, hi, fptr(k)))
    streams = [torch.cuda.Stream(dev) for _ in range(n)]
    torch.cuda.synchronize(dev)
    # each rank's whole run is enqueued on its own stream, one rank after the other: the stream
    # waits on the flags order the slabs on the device (a rank blocked in a wait does not hold
    # the GPU; the others' streams proceed)
    for k, s in enumerate(slabs):
        run_fused(stencil, s, bufs_per_slab[k], T, cfg, links[k], stream=streams[k])
    torch.cuda.synchronize(dev)
    return [b for _, b in bufs_per_slab]


# ---------------------------------------------------------------------------------------------
# bench.py --gpus N (N > 1): one process per GPU under torchrun
# ---------------------------------------------------------------------------------------------
def bench_main(args, workloads):
    """Strong-scaling bench of one workload over N GPUs (see bench.py); rank 0 prints the line."""
    import torch
    import torch.distributed as dist

    import inputs
    import paper_2001_01473_b200 as an5d
    from paper_2001_01473_b200 import perf

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    name, dtype_name, n, T = workloads[args.workload]
    if args.T:
        T = args.T
    dtype = getattr(torch, dtype_name)
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    gext = (n + 2 * rad,) * ndim
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    # the planner picks (bT, vec, h) for this rank's slab shape
    probe = (-(-n // ws) + 2 * rad,) + gext[1:]
    hint = {"bT": args.bt, "vec": args.vec, "h": args.h, "n_thr": getattr(args, "nthr", 0)}
    cfg = st.plan_config(probe, T, hint)
    tuned = False
    if not getattr(args, "no_tune", False):
        # the paper's measured top-5 pick on rank 0, on a grid of one slab's shape;
        # every rank then uses the same (bT, vec, h), which fixes the ghost width of the partition
        pa = an5d.empty_grid(probe, rad, dtype, dev)
        pb = an5d.empty_grid(probe, rad, dtype, dev)
        pa.uniform_()
        st.copy_ring(pa, pb)
        obj = [None]
        if rank == 0:
            t = st.tune(pa, pb, T, hint, top_k=5)
            obj = [{k: t[k] for k in ("bT", "vec", "h", "n_thr", "bS", "direct")}]
        dist.broadcast_object_list(obj, src=0)
        cfg = st.plan_config(probe, T, obj[0])
        tuned = True
        del pa, pb
        torch.cuda.synchronize()
    slabs = partition_aligned(gext[0], rad, ws, cfg["bT"] * rad, int(cfg["h"] or 1))
    s = slabs[rank]
    lext = local_extents(s, gext[1:])
    a = an5d.empty_grid(lext, rad, dtype, dev)
    b = an5d.empty_grid(lext, rad, dtype, dev)
    from bench import fill_uniform, ClockSampler, _peaks
    fill_uniform(a, inputs.DEFAULT_SEED, gext, outer_offset=s.loc_lo)
    b.copy_(a)
    comm = torch.cuda.Stream(dev)
    bufs = [a, b]
    exchange = getattr(args, "exchange", "fused")
    fused = exchange == "fused"
    if exchange == "lib":
        # the library's own NCCL communicator (an5d_set_comm): an5d_run does the whole slab run,
        # ncclSend/ncclRecv of the ghost planes on a library comm stream
        uid = [an5d.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        st.set_comm(uid[0], rank, ws, gext[0], s.loc_lo, s.G)
    if fused:
        # fused halo exchange (NEXT N1): peer-mapped ghost planes written by the sweep kernels
        flag = torch.zeros(32, dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        links, opened = connect_fused(slabs, rank, (a, b), flag)
        links_b, opened_b = links.swapped(), []
        dist.barrier()

    def step(i):
        src, dst = bufs[i % 2], bufs[(i + 1) % 2]
        if fused:
            run_fused(st, s, (src, dst), T, cfg, links if i % 2 == 0 else links_b,
                      stream=torch.cuda.current_stream(dev))
        elif exchange == "lib":
            st.run(src, dst, T, cfg)
        else:
            run_distributed(st, s, (src, dst), T, cfg, comm_stream=comm)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    dist.barrier()
    l0 = st.last_launch_count()
    step(0)
    torch.cuda.synchronize()
    launches_per_step = st.last_launch_count() - l0 + 1   # + the ring copy
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record()
        for i in range(args.steps):
            step(args.warmup + i)
        ev1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # end to end: host (pinned) slab in, owned planes out, every step, max over ranks.  Steps are
    # pipelined over two slab buffer pairs (H2D of step i+1 and D2H of step i-1 overlap the sweeps
    # and exchanges of step i) when a slab is small enough to double-buffer, else serial.
    e2e = None
    if not args.no_e2e:
        n_in = a.untyped_storage().nbytes() // a.element_size()
        flat = lambda t: torch.empty(0, dtype=dtype, device=dev).set_(t.untyped_storage())
        pipelined = a.untyped_storage().nbytes() <= (4 << 30)
        nbuf = 2 if pipelined else 1
        pairs = [(a, b)] + ([(an5d.empty_grid(lext, rad, dtype, dev), an5d.empty_grid(lext, rad, dtype, dev))]
                            if pipelined else [])
        host_in = [torch.empty(n_in, dtype=dtype, pin_memory=True) for _ in range(nbuf)]
        for h_ in host_in:
            h_.copy_(flat(a).cpu())
        owned = [_plane_view(pb, s.out_lo, s.out_hi - s.out_lo) for _, pb in pairs]
        host_out = [torch.empty(owned[0].numel(), dtype=dtype, pin_memory=True) for _ in range(nbuf)]
        main = torch.cuda.current_stream(dev)
        s_in = torch.cuda.Stream(dev) if pipelined else main
        s_out = torch.cuda.Stream(dev) if pipelined else main
        ev_in = [torch.cuda.Event() for _ in range(nbuf)]
        ev_comp = [torch.cuda.Event() for _ in range(nbuf)]
        ev_out = [torch.cuda.Event() for _ in range(nbuf)]
        k_e2e = max(2, min(args.steps, 5))
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        s_in.wait_event(e0)
        s_out.wait_event(e0)
        for i in range(k_e2e):
            j = i % nbuf
            ga, gb = pairs[j]
            if i >= nbuf:
                s_in.wait_event(ev_comp[j])
            with torch.cuda.stream(s_in):
                flat(ga).copy_(host_in[j], non_blocking=True)
            ev_in[j].record(s_in)
            main.wait_event(ev_in[j])
            if i >= nbuf:
                main.wait_event(ev_out[j])
            if fused:
                # the e2e pairs are other buffers: the exchange for them goes through the NCCL
                # runner (the fused links map the timed buffers a, b only)
                run_distributed(st, s, (ga, gb), T, cfg, comm_stream=comm)
            elif exchange == "lib":
                st.run(ga, gb, T, cfg)
            else:
                run_distributed(st, s, (ga, gb), T, cfg, comm_stream=comm)
            ev_comp[j].record(main)
            s_out.wait_event(ev_comp[j])
            with torch.cuda.stream(s_out):
                host_out[j].copy_(owned[j], non_blocking=True)
            ev_out[j].record(s_out)
        for j in range(nbuf):
            main.wait_event(ev_out[j])
        e1.record(main)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / k_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        nb = torch.tensor([float(n_in * a.element_size()), float(host_out[0].numel() * a.element_size())],
                          dtype=torch.float64, device=dev)
        dist.all_reduce(nb)
        e2e = {"value": round(float(n) ** ndim * T / (float(te.item()) * 1e-3) / 1e9, 3), "unit": "GCells/s",
               "h2d_bytes_per_step": int(nb[0].item()), "d2h_bytes_per_step": int(nb[1].item()),
               "ms_per_step": round(float(te.item()), 3), "steps": k_e2e, "pipelined": pipelined}
        del pairs
    cells = float(n) ** ndim
    gcells = cells * T / (ms * 1e-3) / 1e9
    F = perf.flops_per_cell(ndim, rad, shape, div != 1.0)
    rl = None
    if rank == 0:
        # step-level roofline per GPU (the whole step incl. the halo exchange, rank 0's slab): the
        # algorithmic bytes of SURVEY 8(d) at the run schedule's effective stream-block length
        try:
            geom = st.describe(lext, cfg)
            nbd = ndim - 1
            ntiles = geom["n_tiles"][0] * (geom["n_tiles"][1] if ndim == 3 else 1)
            h_eff = ntiles * (lext[0] - 2 * rad) / max(1, geom["n_units"])
            peaks = _peaks()
            elem = 4 if dtype == torch.float32 else 8
            roof = perf.roofline(ndim=ndim, rad=rad, shape=shape, has_div=div != 1.0, dtype_bytes=elem,
                                 bT=cfg["bT"], tile_loaded=geom["bS_loaded"][:nbd], tile_compute=geom["compute"][:nbd],
                                 h=h_eff, hbm_gbs=peaks["hbm_gbs"],
                                 fp_peak=perf.fp_peak_flops(elem, 148, peaks.get("sm_max_mhz") or 1965.0))
            ach = roof["alg_bytes_per_cell_step"] * (float(n) ** ndim * T / ws) / (ms * 1e-3) / 1e9
            rl = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                  "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": None,
                  "basis": "whole step per GPU (sweeps + NCCL halo exchange), rank 0's slab",
                  "R_read": round(roof["R_read"], 4)}
        except Exception as e:  # the line is still printed; say why the roofline is missing
            rl = {"error": str(e)[:200]}
        clocks = clk.summary()
        line = {
            "metric": f"GCells/s ({name} {dtype_name} {n}^{ndim}, T={T})", "value": round(gcells, 3),
            "unit": "GCells/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if dtype == torch.float32 else "f64", "data": "synthetic",
            "config": {"workload": args.workload, "stencil": name, "grid": list(gext), "T": T, "bT": cfg["bT"],
                       "vec": cfg["vec"], "h": cfg["h"], "n_thr": cfg.get("n_thr"),
                       "parallelism": f"slab{ws} (outermost dim, " + ("fused peer-store halo exchange over NVLink)" if fused else
                                                                      ("library NCCL halo, an5d_set_comm)" if exchange == "lib" else "NCCL halo)")),
                       "planner": "model top-5, measured pick on rank 0 (P:784-793)" if tuned else "model",
                       "l2": "inputs larger than L2"},
            "gflops": round(gcells * F, 2), "roofline": rl, "cpu_baseline": None, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps * ws,
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"]},
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    if fused:
        for base in opened + opened_b:
            an5d.ipc_close(base)
    dist.destroy_process_group()
    return 0
