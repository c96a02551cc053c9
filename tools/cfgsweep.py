"""Explore blocking configurations: time sweeps of one stencil for every (bT, vec, h[, direct]) given.

usage: cfgsweep.py NAME DTYPE [bT list] [vec list] [h list] [direct list] [n sweeps]
   e.g. cfgsweep.py star3d1r f32 1,2,3,4 2,4 32,64,128 0 6
Prints one JSON line per configuration: sweep-only GCells/s (interior cells x degree / sweep time)
and the planner's model time for the same configuration.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import inputs
import paper_2001_01473_b200 as an5d
from bench import fill_uniform

name, dt = sys.argv[1], sys.argv[2]
lst = lambda i, d: [int(v) for v in (sys.argv[i] if len(sys.argv) > i else d).split(",")]
bts, vecs, hs, directs = lst(3, "1,2,3,4"), lst(4, "2,4"), lst(5, "0"), lst(6, "0")
n = int(sys.argv[7]) if len(sys.argv) > 7 else 6
dtype = torch.float32 if dt == "f32" else torch.float64
ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
size = 16384 if ndim == 2 else 512
ext = (size + 2 * rad,) * ndim
st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
a = an5d.empty_grid(ext, rad, dtype)
b = an5d.empty_grid(ext, rad, dtype)
fill_uniform(a, 1, ext)
b.copy_(a)
st.copy_ring(a, b)
cells = float(size) ** ndim
print(json.dumps({"planner": st.plan_config(ext, 1000)}), flush=True)
for direct in directs:
    for vec in vecs:
        for bt in bts:
            for h in hs:
                try:
                    cfg = st.plan_config(ext, 1000, {"bT": bt, "h": h, "vec": vec, "direct": direct})
                    geo = st.describe(ext, cfg)
                except an5d.AN5DError as e:
                    continue
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
                for i in range(2):
                    st.sweep(a if i % 2 == 0 else b, b if i % 2 == 0 else a, bt, cfg)
                torch.cuda.synchronize()
                ev[0].record()
                for i in range(n):
                    st.sweep(a if i % 2 == 0 else b, b if i % 2 == 0 else a, bt, cfg)
                    ev[i + 1].record()
                torch.cuda.synchronize()
                ms = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(n))
                med = ms[len(ms) // 2]
                print(json.dumps({"name": name, "dt": dt, "bT": bt, "vec": vec, "h": cfg["h"], "direct": direct,
                                  "ms": round(med, 4), "gcells": round(cells * bt / med / 1e6, 1),
                                  "regs": geo["regs_per_thread"], "smem": geo["smem_bytes"],
                                  "blocks": geo["grid_blocks"]}), flush=True)
