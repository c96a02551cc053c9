"""Run N sweeps of one 2D/3D stencil configuration (for ncu captures):
sweeponly.py name dtype bT h vec n [n_thr [bS_y]]  (3D bS_y: the loaded tile height naming a layout)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs, paper_2001_01473_b200 as an5d
from bench import fill_uniform
name, dt, bt, h, vec, n = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6])
dtype = torch.float32 if dt == "f32" else torch.float64
ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
size = 16384 if ndim == 2 else 512
ext = (size + 2 * rad,) * ndim
st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
nthr = int(sys.argv[7]) if len(sys.argv) > 7 else 0
hint = {"bT": bt, "h": h, "vec": vec, "n_thr": nthr}
if len(sys.argv) > 8:
    hint["bS"] = [int(sys.argv[8]), 0]
cfg = st.plan_config(ext, 1000, hint)
print(cfg, file=sys.stderr)
a = an5d.empty_grid(ext, rad, dtype); b = an5d.empty_grid(ext, rad, dtype)
fill_uniform(a, 1, ext); b.copy_(a)
st.copy_ring(a, b)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
import time
ev[0].record()
host = []
for i in range(n):
    t0 = time.perf_counter()
    st.sweep(a if i % 2 == 0 else b, b if i % 2 == 0 else a, cfg["bT"], cfg)
    host.append(round((time.perf_counter() - t0) * 1e3, 3))
    ev[i + 1].record()
torch.cuda.synchronize()
print("host ms", host, file=sys.stderr)
print("sweep ms", [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(n)], file=sys.stderr)
