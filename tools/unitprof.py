"""Debug: per-unit timing of one 2D sweep (AN5D_UNIT_PROFILE), summarised per unit class."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2001_01473_b200 as an5d
from bench import fill_uniform

name = sys.argv[1] if len(sys.argv) > 1 else "star2d1r"
bt = int(sys.argv[2]) if len(sys.argv) > 2 else 8
h = int(sys.argv[3]) if len(sys.argv) > 3 else 0
vec = int(sys.argv[4]) if len(sys.argv) > 4 else 0
n = 16384
ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
ext = (n + 2 * rad,) * 2
st = an5d.Stencil(ndim, rad, shape, tab, div, torch.float32)
cfg = st.plan_config(ext, 1000, {"bT": bt, "h": h, "vec": vec})
print(cfg)
a = an5d.empty_grid(ext, rad); b = an5d.empty_grid(ext, rad)
fill_uniform(a, 1, ext); b.copy_(a)
for _ in range(3):
    st.sweep(a, b, bt, cfg)
torch.cuda.synchronize()
path = "gpurun_out/unitprof.txt"
if os.path.exists(path): os.remove(path)
os.environ["AN5D_UNIT_PROFILE"] = path
st.sweep(a, b, bt, cfg)
torch.cuda.synchronize()
del os.environ["AN5D_UNIT_PROFILE"]
rows = [l.split() for l in open(path) if not l.startswith("#")]
hdr = open(path).readline()
print(hdr)
u = np.array([[int(x) for x in r] for r in rows])
t0 = u[:, 1].min()
dur = (u[:, 2] - u[:, 1]) / 1e3
ntx = int(hdr.split("ntx")[1].split()[0])
tile = u[:, 0] % ntx; sb = u[:, 0] // ntx
print("total us", (u[:, 2].max() - t0) / 1e3, "unit us mean/min/max", dur.mean(), dur.min(), dur.max())
nxe = 3 if ntx >= 4 else ntx
xe = u[:, 0] < nxe * (u[:, 0].max() + 1) // ntx; ye = ~xe & (u[:, 0] < nxe * ((u[:, 0].max() + 1) // ntx) + 2 * (ntx - nxe))
for nm, m in [("interior", ~xe & ~ye), ("xedge", xe & ~ye), ("yedge", ye & ~xe), ("corner", xe & ye)]:
    if m.any(): print(nm, m.sum(), "mean us", dur[m].mean(), "max", dur[m].max())
print("start spread us", (u[:, 1].max() - t0) / 1e3)
per_sm = collections.Counter(u[:, 3])
print("units per SM: min", min(per_sm.values()), "max", max(per_sm.values()), "n SMs", len(per_sm))
sm_end = collections.defaultdict(int)
for r in u: sm_end[r[3]] = max(sm_end[r[3]], r[2] - t0)
e = np.array(list(sm_end.values())) / 1e3
print("SM finish us min/median/max", e.min(), np.median(e), e.max())
slow = np.argsort(-dur)[:10]
for i in slow: print("slow unit", u[i, 0], "tile", tile[i], "sb", sb[i], "sm", u[i, 3], "us", dur[i], "start", (u[i,1]-t0)/1e3)
