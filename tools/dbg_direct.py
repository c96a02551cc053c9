import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import inputs, oracle, paper_2001_01473_b200 as an5d
for name, dtype in [("box2d1r", torch.float32), ("box2d2r", torch.float32), ("box2d1r", torch.float64)]:
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = (61 + 2 * rad, 411 + 2 * rad)
    g = inputs.global_grid(inputs.DEFAULT_SEED, ext)
    npdt = np.float32 if dtype == torch.float32 else np.float64
    st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
    for vec in (4, 8):
        for bT in (1, 2, 3, 5):
            for direct in (0, 1):
                cfg = {"bT": bT, "vec": vec, "h": 16, "direct": direct}
                try:
                    st.describe(ext, cfg)
                except an5d.AN5DError as e:
                    continue
                a = an5d.to_grid(torch.from_numpy(g.astype(npdt)).cuda(), rad)
                b = an5d.empty_grid(ext, rad, dtype); b.fill_(float("nan"))
                wc = torch.zeros(ext, dtype=torch.int32, device="cuda")
                st.copy_ring(a, b)
                st.sweep(a, b, bT, cfg, write_count=wc)
                torch.cuda.synchronize()
                got = b.cpu().numpy(); w = wc.cpu().numpy()
                exp = oracle.run(g, rad, shape, tab, div, bT, npdt)
                core = (slice(rad, ext[0] - rad), slice(rad, ext[1] - rad))
                bad = ~np.isclose(got, exp, rtol=1e-4, atol=1e-5)
                bad[~np.ones_like(bad)] = False
                wb = (w[core] != 1)
                ys, xs = np.nonzero(bad)
                print(name, dtype, cfg, "bad", bad[core].sum(), "nan", np.isnan(got[core]).sum(), "wc!=1", wb.sum(),
                      "rows", sorted(set(ys.tolist()))[:12], "cols", sorted(set(xs.tolist()))[:12], flush=True)
