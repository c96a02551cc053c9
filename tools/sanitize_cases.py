"""Small runs of every kernel family through the C ABI, for compute-sanitizer (racecheck /
synccheck / memcheck): 2D one warp per tile and the two-warp level split, 3D 256- and 512-thread
layouts (TMA + mbarrier staging, shared-memory halo exchange), the fp32 box rad-4 runtime plane
loop, the fused halo exchange in one process, and (round 2) thread-block clusters, output-
stationary / staged-halo 3D tiles, gradient2d and a multi-field system.  Each result is checked
against the oracle.

usage (under gpurun): compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import inputs
import oracle
import paper_2001_01473_b200 as an5d
from paper_2001_01473_b200 import slab

CASES = [
    ("star2d1r", torch.float32, (29, 600), 9, {"bT": 4, "vec": 8, "h": 8, "n_thr": 32}),
    ("star2d1r", torch.float32, (29, 600), 9, {"bT": 4, "vec": 8, "h": 8, "n_thr": 64}),
    ("box2d2r", torch.float64, (21, 300), 5, {"bT": 2, "vec": 4, "h": 8}),
    ("box2d2r", torch.float32, (21, 600), 5, {"bT": 2, "vec": 8, "h": 8, "direct": 1}),
    ("star3d1r", torch.float32, (13, 40, 140), 7, {"bT": 3, "vec": 2, "h": 4, "n_thr": 256}),
    ("star3d1r", torch.float64, (13, 40, 140), 7, {"bT": 3, "vec": 2, "h": 4, "n_thr": 512}),
    ("box3d4r", torch.float32, (9, 40, 130), 2, {"bT": 1, "vec": 2, "h": 4}),
    # round 2: clusters (DSMEM halo sharing, split cluster barrier), output-stationary and
    # y/x-staged tiles, gradient2d, the level split with uniform scheduling
    ("star3d1r", torch.float32, (13, 80, 140), 7, {"bT": 3, "vec": 2, "h": 4, "n_thr": 256, "bS": [64, 0]}),
    ("star3d1r", torch.float64, (13, 80, 140), 7, {"bT": 3, "vec": 2, "h": 4, "n_thr": 512, "bS": [64, 0]}),
    ("box3d3r", torch.float32, (9, 40, 130), 2, {"bT": 1, "vec": 2, "h": 4, "n_thr": 256, "bS": [38, 70]}),
    ("star3d2r", torch.float32, (13, 40, 140), 5, {"bT": 2, "vec": 2, "h": 4, "n_thr": 256, "bS": [36, 0]}),
    ("star3d1r", torch.float64, (13, 40, 140), 7, {"bT": 3, "vec": 2, "h": 4, "n_thr": 512, "bS": [34, 66]}),
    ("gradient2d", torch.float32, (29, 600), 7, {"bT": 3, "vec": 8, "h": 8}),
]


def rel(got, exp, rad):
    core = tuple(slice(rad, e - rad) for e in exp.shape)
    return float(np.abs(got[core] - exp[core]).max() / np.abs(exp[core]).max())


def main():
    torch.cuda.set_device(0)
    for name, dt, n_int, T, cfg in CASES:
        ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
        ext = tuple(v + 2 * rad for v in n_int)
        g = inputs.global_grid(5, ext)
        npdt = np.float32 if dt == torch.float32 else np.float64
        st = an5d.Stencil(ndim, rad, shape, tab, div, dt)
        a = an5d.to_grid(torch.from_numpy(g.astype(npdt)).cuda(), rad)
        b = an5d.empty_grid(ext, rad, dt)
        st.run(a, b, T, cfg)
        torch.cuda.synchronize()
        err = rel(b.cpu().numpy(), oracle.run(g, rad, shape, tab, div, T, npdt), rad)
        print(f"{name} {dt} {cfg}: rel_linf {err:.2e}", flush=True)
        assert err <= (1e-5 if dt == torch.float32 else 1e-12)
    # multi-field system (2 fields, one kernel)
    ndim, rad, shape, nf, tab = inputs.system_problem("star2d1r-x2")
    ext = (31, 602)
    f = inputs.system_fields(5, nf, ext)
    sy = an5d.System(ndim, rad, shape, tab, torch.float32)
    a = an5d.to_fields(torch.from_numpy(f.astype(np.float32)).cuda(), rad)
    b = an5d.empty_fields(nf, ext, rad, torch.float32)
    sy.run(a, b, 9, {"bT": 3, "vec": 8, "h": 8})
    torch.cuda.synchronize()
    exp = oracle.run_system(f, rad, shape, tab, 9, np.float32)
    err = float(np.abs(b.cpu().numpy() - exp).max() / np.abs(exp).max())
    print(f"star2d1r-x2 float32: rel_linf {err:.2e}", flush=True)
    assert err <= 1e-5
    # fused halo exchange, 3 slabs on one device
    ndim, rad, shape, tab, div = inputs.benchmark_problem("star2d1r")
    gext = (62 + 2 * rad, 300 + 2 * rad)
    g = inputs.global_grid(9, gext)
    st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
    cfg = st.plan_config(gext, 9, {"bT": 3, "h": 8, "vec": 8})
    parts = slab.partition(gext[0], rad, 3, 3 * rad)
    bufs = [(an5d.to_grid(torch.from_numpy(g[s.loc_lo:s.loc_hi].astype(np.float32)).cuda(), rad),
             an5d.empty_grid((s.n_local,) + gext[1:], rad, torch.float32)) for s in parts]
    outs = slab.loopback_fused(st, parts, bufs, 9, cfg)
    got = np.concatenate([o.cpu().numpy()[s.out_lo:s.out_hi] for s, o in zip(parts, outs)])
    exp = oracle.run(g, rad, shape, tab, div, 9, np.float32)[rad:gext[0] - rad]
    err = float(np.abs(got - exp).max() / np.abs(exp).max())
    print(f"fused loopback 3 slabs: rel_linf {err:.2e}", flush=True)
    assert err <= 1e-5
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
