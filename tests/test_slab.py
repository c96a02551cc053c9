"""Multi-GPU slab decomposition: host bookkeeping and the exchange protocol.

* Pure partition / sweep-split invariants (no process group).
* world_size 2 (and 3) ``gloo`` runs on CPU of the SAME runner the GPU bench uses
  (slab.run_distributed), with the oracle standing in for the per-slab sweep (tests may call the
  oracle; the product path calls an5d_sweep).  The gathered owned planes must equal the oracle on
  the whole global grid bit-for-bit: the per-cell arithmetic does not depend on the slab split.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle
from paper_2001_01473_b200 import slab


def test_partition_covers_interior_disjointly():
    for gE0, rad, n, G in [(1540, 2, 8, 6), (518, 3, 4, 9), (40, 1, 3, 4), (23, 1, 2, 3)]:
        parts = slab.partition(gE0, rad, n, G)
        owned = []
        for s in parts:
            owned += list(range(s.own_lo, s.own_hi))
            assert s.loc_lo == max(0, s.own_lo - G) and s.loc_hi == min(gE0, s.own_hi + G)
            assert s.own_hi - s.own_lo >= G
        assert owned == list(range(rad, gE0 - rad))


def test_partition_aligned_to_stream_blocks():
    """Owned chunks are multiples of h where that leaves every rank >= G planes,
    else the plain split; both cover the interior disjointly."""
    for gE0, rad, n, G, h in [(1540, 2, 8, 6, 64), (1540, 2, 4, 6, 78), (518, 3, 4, 9, 100), (40, 1, 3, 4, 16)]:
        parts = slab.partition_aligned(gE0, rad, n, G, h)
        owned = []
        for s in parts:
            owned += list(range(s.own_lo, s.own_hi))
        assert owned == list(range(rad, gE0 - rad))
        chunks = [s.own_hi - s.own_lo for s in parts]
        if all(c % h == 0 for c in chunks[:-1]):
            assert min(chunks) >= G
    assert all((s.own_hi - s.own_lo) % 64 == 0 for s in slab.partition_aligned(1540, 2, 8, 6, 64)[:-1])


def test_partition_rejects_thin_slabs():
    with pytest.raises(ValueError):
        slab.partition(20, 1, 8, 6)


def test_sweep_parts_exchange_is_symmetric():
    """Every receive has a matching send of the same length on the peer, and received ghosts lie
    outside the owned planes but inside the local array; boundary + interior tile the owned planes."""
    for gE0, rad, n, G, h in [(1540, 2, 8, 6, 64), (100, 1, 4, 4, 8), (60, 2, 3, 8, 100)]:
        parts = slab.partition(gE0, rad, n, G)
        for nd in range(0, G // rad + 1):
            sp = [slab.sweep_parts(s, nd, h) for s in parts]
            for s, p in zip(parts, sp):
                cover = sorted(p.boundary + p.interior)
                assert cover[0][0] == s.out_lo and cover[-1][1] == s.out_hi
                assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
                for peer, lo, m in p.recvs:
                    assert m == nd * rad
                    assert (lo + m <= s.out_lo) or (lo >= s.out_hi)
                    assert 0 <= lo and lo + m <= s.n_local
                    (snd,) = [x for x in sp[peer].sends if x[0] == s.rank]
                    assert snd[2] == m
                    # the sent planes are the same global planes as the received ghosts
                    assert parts[peer].loc_lo + snd[1] == s.loc_lo + lo
                # sent planes are owned and produced by the boundary part
                for peer, lo, m in p.sends:
                    assert s.out_lo <= lo and lo + m <= s.out_hi
                    assert any(b0 <= lo and lo + m <= b1 for b0, b1 in p.boundary)


class OracleSlabStencil:
    """Test stand-in for Stencil on CPU tensors: the oracle advances the whole local slab (its
    local faces act as Dirichlet planes, which only corrupts cells within d*rad of a ghost face:
    exactly the cone the owned planes never see)."""

    def __init__(self, rad, shape, tab, div, npdt):
        self.rad, self.shape, self.tab, self.div, self.npdt = rad, shape, tab, div, npdt

    def copy_ring(self, a, b, outer_offset=0, global_outer_extent=None):
        r = self.rad
        g = global_outer_extent
        an, bn = a.numpy(), b.numpy()
        for z in range(a.shape[0]):
            gz = z + outer_offset
            if gz < r or gz >= g - r:
                bn[z] = an[z]
            else:
                m = np.ones(an.shape[1:], bool)
                m[tuple(slice(r, e - r) for e in an.shape[1:])] = False
                bn[z][m] = an[z][m]

    def sweep(self, src, dst, d, cfg, outer_offset=0, global_outer_extent=None, out_lo=None, out_hi=None):
        res = oracle.run(src.numpy(), self.rad, self.shape, self.tab, self.div, d, self.npdt)
        dst.numpy()[out_lo:out_hi] = res[out_lo:out_hi]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, case, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    name, n_int, T, bT, h, dt = case
    npdt = np.float32 if dt == "f32" else np.float64
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    gext = tuple(v + 2 * rad for v in n_int)
    s = slab.partition(gext[0], rad, ws, bT * rad)[rank]
    lext = slab.local_extents(s, gext[1:])
    loc = inputs.global_grid(7, lext, outer_offset=s.loc_lo, global_extents=gext).astype(npdt)
    a = torch.from_numpy(loc.copy())
    b = torch.full(lext, float("nan"), dtype=a.dtype)
    st = OracleSlabStencil(rad, shape, tab, div, npdt)
    res = slab.run_distributed(st, s, (a, b), T, {"bT": bT, "h": h})
    np.save(os.path.join(out_dir, f"r{rank}.npy"), res.numpy()[s.out_lo:s.out_hi])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case,ws", [
    (("star2d1r", (37, 29), 9, 4, 4, "f32"), 2),      # schedule 4,4,1 (odd count)
    (("box2d2r", (41, 23), 6, 3, 2, "f64"), 2),       # 3,3 -> split 3,2,1
    (("star3d2r", (30, 9, 11), 5, 2, 3, "f32"), 2),   # 2,2,1
    (("j3d27pt", (25, 8, 9), 4, 1, 1, "f64"), 3),     # bT = 1, even T -> trailing copy
    (("star2d3r", (60, 19), 7, 2, 50, "f32"), 3),     # h larger than a slab: no overlap split
])
def test_gloo_slab_run_matches_global_oracle(tmp_path, case, ws):
    port = _free_port()
    mp.spawn(_worker, args=(ws, port, case, str(tmp_path)), nprocs=ws, join=True)
    name, n_int, T, bT, h, dt = case
    npdt = np.float32 if dt == "f32" else np.float64
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    gext = tuple(v + 2 * rad for v in n_int)
    g = inputs.global_grid(7, gext).astype(npdt)
    exp = oracle.run(g, rad, shape, tab, div, T, npdt)
    got = np.concatenate([np.load(os.path.join(tmp_path, f"r{k}.npy")) for k in range(ws)])
    assert np.array_equal(got, exp[rad:gext[0] - rad])
