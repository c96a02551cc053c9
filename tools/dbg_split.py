"""Debug: run small 2D grids through chosen configurations (compute-sanitizer target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, oracle, paper_2001_01473_b200 as an5d
cases = [("star2d1r", torch.float32, {"bT": 2, "vec": 8, "h": 16, "n_thr": 64}),
         ("box2d1r", torch.float32, {"bT": 4, "vec": 8, "h": 16, "n_thr": 64}),
         ("star2d1r", torch.float32, {"bT": 7, "vec": 8, "h": 16, "n_thr": 64})]
for name, dt, cfg in cases:
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = (int(os.environ.get("NY", 61)) + 2 * rad, int(os.environ.get("NX", 700)) + 2 * rad)
    g = inputs.global_grid(1, ext)
    st = an5d.Stencil(ndim, rad, shape, tab, div, dt)
    a = an5d.to_grid(torch.from_numpy(g.astype(np.float32)).cuda(), rad)
    b = an5d.empty_grid(ext, rad, dt)
    T = 2 * cfg["bT"] + 1
    print(name, st.plan_config(ext, T, cfg), flush=True)
    st.run(a, b, T, cfg)
    torch.cuda.synchronize()
    exp = oracle.run(g, rad, shape, tab, div, T, np.float32)
    print(name, cfg, "maxerr", float(np.abs(b.cpu().numpy() - exp).max()), flush=True)
