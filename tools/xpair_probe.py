"""Each XPAIR 3D case in its own process (a sticky CUDA error cannot mask the others):
python tools/xpair_probe.py  -> one line per case: OK / error / max rel err vs oracle."""
import os, subprocess, sys
CASES = [("box3d1r", 2, 32), ("box3d1r", 2, 34), ("star3d1r", 2, 32), ("star3d1r", 2, 64), ("star3d2r", 1, 32),
         ("box3d2r", 1, 32), ("box3d2r", 1, 36), ("j3d27pt", 2, 64), ("star3d1r", 3, 32)]
CHILD = r'''
import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import inputs, oracle, paper_2001_01473_b200 as an5d
name, bT, bsy = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
ext = (23 + 2 * rad, 131 + 2 * rad, 509 + 2 * rad)
g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
cfg = {"bT": bT, "vec": 2, "h": 8, "n_thr": 256, "bS": [bsy, 0]}
d = st.describe(ext, cfg)
a = an5d.to_grid(torch.from_numpy(g.astype(np.float32)).cuda(), rad)
b = an5d.empty_grid(ext, rad, torch.float32)
st.run(a, b, bT, cfg)
torch.cuda.synchronize()
got = b.cpu().numpy(); exp = oracle.run(g, rad, shape, tab, div, bT, np.float32)
core = tuple(slice(rad, e - rad) for e in ext)
print("halo", d["halo_loaded"], "compute", d["compute"], "err", float(np.abs(got[core] - exp[core]).max() / np.abs(exp[core]).max()))
'''
for c in CASES:
    r = subprocess.run([sys.executable, "-c", CHILD] + [str(v) for v in c], capture_output=True, text=True,
                       env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"), timeout=300)
    tail = (r.stdout.strip().splitlines() or [""])[-1] if r.returncode == 0 else r.stderr.strip().splitlines()[-1]
    print(c, "rc", r.returncode, tail, flush=True)
