#!/usr/bin/env python
"""bench.py -- AN5D N.5D stencil sweep on B200: GCells/s and GFLOP/s, roofline fraction, CPU oracle.

Driver contract: `python bench.py --gpus N --steps K --warmup W` (N > 1 under torchrun, one rank per
GPU, NCCL) prints ONE JSON line on rank 0.  A "step" is one full an5d_run of the workload: ring copy
plus every N.5D sweep of T = 1000 time steps (all hot-path rows of SURVEY.md §8(a)) on one grid.

Default workload (BASELINE.json configs[1], its headline row = PAPER.md Table 5 row 1):
star2d1r, fp32, 16384^2 interior, T = 1000, b_T / tile / stream block from the host planner.
Inputs: seeded synthetic (inputs.uniform24, dyadic coefficients summing to 1), resident in HBM.
L2: each grid buffer is 1 GiB > 126 MB L2, so every sweep streams from HBM (no flush needed).

`--impl reference` times the CPU oracle (oracle/, the plain double-buffered loop) as the reference
arm on the same workload: each step is a bounded sample (the full grid for a few time steps).
`--suite` runs the BASELINE configs 2-3 b_T sweeps and writes profiles/suite.json (not a driver line).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOADS = {
    # name: (stencil, dtype, interior size per dim, T)
    "star2d1r-f32-16384": ("star2d1r", "float32", 16384, 1000),
}
for _n in ("star2d1r", "star2d2r", "star2d3r", "star2d4r", "box2d1r", "box2d2r", "box2d3r", "box2d4r",
           "j2d5pt", "j2d9pt", "j2d9pt-gol", "gradient2d"):
    for _dt in ("f32", "f64"):
        WORKLOADS[f"{_n}-{_dt}-16384"] = (_n, "float32" if _dt == "f32" else "float64", 16384, 1000)
for _n in ("star3d1r", "star3d2r", "star3d3r", "star3d4r", "box3d1r", "box3d2r", "box3d3r", "box3d4r",
           "j3d27pt"):
    for _dt in ("f32", "f64"):
        WORKLOADS[f"{_n}-{_dt}-512"] = (_n, "float32" if _dt == "f32" else "float64", 512, 1000)
WORKLOADS["star3d2r-f32-1536"] = ("star3d2r", "float32", 1536, 1000)
# multi-field systems (NEXT N4): GCells/s counts cells of every field
for _n in ("star2d1r-x2", "box2d1r-x2"):
    for _dt in ("f32", "f64"):
        WORKLOADS[f"{_n}-{_dt}-16384"] = (_n, "float32" if _dt == "f32" else "float64", 16384, 1000)
DEFAULT = "star2d1r-f32-16384"


def _peaks():
    p = {"hbm_gbs": None, "source": None}
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        p.update(hbm_gbs=d.get("hbm_gbs"), sm_max_mhz=d.get("sm_max_mhz"), source="measured")
    if not p["hbm_gbs"]:
        p.update(hbm_gbs=6650.0, sm_max_mhz=1965.0, source="fallback")   # B200_PROFILING.md fallback
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        time.sleep(0.25)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _traffic(workload, cfg):
    """DRAM bytes per launch of the dominant kernel (dram__bytes_read.sum + dram__bytes_write.sum)
    from a committed ncu --set full capture of the same workload (profiles/traffic.json, entries
    written by tools/ncu_summary.py).  Exact (b_T, vec, h) match first; else the capture of the same
    (b_T, vec) with the nearest h, labelled as such in traffic_source (the DRAM bytes depend on h
    only through the stream-block overlap, 2 b_T rad / h); else None."""
    path = os.path.join(REPO, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        ents = json.load(f).get(workload)
    if not ents:
        return None
    if isinstance(ents, dict):
        ents = [ents]
    same = [e for e in ents if e.get("bT") == cfg.get("bT") and e.get("vec") == cfg.get("vec")]
    if not same:
        return None
    e = min(same, key=lambda e: abs(e.get("h", 0) - cfg.get("h", 0)))
    note = "" if e.get("h") == cfg.get("h") else f"; nearest h to this run's h {cfg.get('h')}"
    src = e.get("profile") or e.get("source", "ncu")
    return {"traffic_bytes": e["traffic_bytes"], "source": f"{src} (bT {e['bT']}, vec {e['vec']}, h {e['h']}{note})"}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def fill_uniform(t, seed, global_extents, outer_offset=0):
    """Fill a (possibly strided) grid view with inputs.uniform24 keyed by GLOBAL linear index,
    generated on the device plane by plane (plumbing; same values as the numpy generator)."""
    import torch
    import inputs
    inner = 1
    for e in global_extents[1:]:
        inner *= e
    per = max(1, (1 << 24) // inner)
    for z0 in range(0, t.shape[0], per):
        z1 = min(t.shape[0], z0 + per)
        lin = (torch.arange(z0 + outer_offset, z1 + outer_offset, device=t.device, dtype=torch.int64)[:, None] * inner
               + torch.arange(inner, device=t.device, dtype=torch.int64)[None, :])
        v = inputs.uniform24_torch(seed, lin).to(t.dtype).reshape((z1 - z0,) + tuple(global_extents[1:]))
        t[z0:z1].copy_(v)


def cpu_oracle_rate(name, dtype_name, n, host_grid, budget_s=12.0, max_T=None):
    """Time the oracle (as it stands) on the box's host cores on a bounded sample of the workload:
    the full grid for T_cpu time steps, T_cpu calibrated so the run takes about `budget_s`."""
    import numpy as np
    import inputs
    import oracle
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    npdt = np.float32 if dtype_name == "float32" else np.float64
    g = np.ascontiguousarray(host_grid, dtype=npdt)
    cells = float(n) ** ndim
    nt = oracle.max_threads()
    oracle.run(g, rad, shape, tab, div, 1, npdt, nthreads=nt)           # warm (page-in, threads)
    t0 = time.perf_counter()
    oracle.run(g, rad, shape, tab, div, 2, npdt, nthreads=nt)
    t1 = (time.perf_counter() - t0) / 2                                  # seconds per time step
    T_cpu = max(1, int(budget_s / max(t1, 1e-6)))
    if max_T:
        T_cpu = min(T_cpu, max_T)
    t0 = time.perf_counter()
    oracle.run(g, rad, shape, tab, div, T_cpu, npdt, nthreads=nt)
    dt = time.perf_counter() - t0
    return {"value": cells * T_cpu / dt / 1e9, "unit": "GCells/s", "cores": nt, "kind": "oracle",
            "sample": f"{name} {dtype_name} full {n}^{ndim} grid, {T_cpu} of 1000 time steps "
                      f"(naive double-buffered C loop, OpenMP {nt} threads, {dt:.1f} s)",
            "seconds": dt, "T_sample": T_cpu}


def table2_flops_per_cell(ndim, rad, shape, has_div):
    """PAPER.md Table 2 FLOP/cell: k taps -> 2k-1 FLOPs, +1 for the /c_0 of the
    j-stencils; gradient2d 19.  Computed here so the reference arm loads nothing from
    the product package."""
    if shape == 2:
        return 19
    k = (2 * rad + 1) ** ndim if shape == 1 else 2 * ndim * rad + 1
    return 2 * k - 1 + (1 if has_div else 0)


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only at N>1)."""
    import numpy as np
    import inputs
    import oracle
    ws, rank, _ = _dist()
    if ws > 1 and rank != 0:
        return 0
    name, dtype_name, n, T = WORKLOADS[args.workload]
    ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
    ext = (n + 2 * rad,) * ndim
    npdt = np.float32 if dtype_name == "float32" else np.float64
    try:
        import torch
        if torch.cuda.is_available():
            t = torch.empty(ext, dtype=torch.float64, device="cuda")
            fill_uniform(t, inputs.DEFAULT_SEED, ext)
            g = t.cpu().numpy().astype(npdt)
            del t
        else:
            raise RuntimeError
    except Exception:
        g = inputs.global_grid(inputs.DEFAULT_SEED, ext).astype(npdt)
    nt = oracle.max_threads()
    oracle.run(g, rad, shape, tab, div, 1, npdt, nthreads=nt)          # warm (page-in, threads)
    t0 = time.perf_counter()
    oracle.run(g, rad, shape, tab, div, 2, npdt, nthreads=nt)
    t1 = (time.perf_counter() - t0) / 2                                  # seconds per time step
    per_step = max(1, int(args.ref_step_seconds / max(t1, 1e-6)))
    for _ in range(args.warmup):
        oracle.run(g, rad, shape, tab, div, per_step, npdt, nthreads=nt)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.run(g, rad, shape, tab, div, per_step, npdt, nthreads=nt)
        times.append(time.perf_counter() - t0)
    cells = float(n) ** ndim
    tot = sum(times)
    val = cells * per_step * args.steps / tot / 1e9
    F = table2_flops_per_cell(ndim, rad, shape, div != 1.0)
    line = {
        "impl": "reference", "metric": f"GCells/s ({name} {dtype_name} {n}^{ndim}, T={T})", "value": round(val, 4),
        "unit": "GCells/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot / args.steps, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if dtype_name == "float32" else "f64", "data": "synthetic",
        "config": {"workload": args.workload, "stencil": name, "grid": list(ext), "T": T,
                   "step": f"{per_step} time steps of the full grid (bounded sample of the T={T} run)"},
        "gflops": round(val * F, 3),
        "cpu_baseline": {"value": round(val, 4), "unit": "GCells/s", "cores": nt, "kind": "oracle",
                         "sample": f"full grid, {per_step} time steps per step, {args.steps} steps"},
        "e2e": {"value": round(val, 4), "unit": "GCells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="an5d", choices=["an5d", "reference"])
    ap.add_argument("--workload", default=DEFAULT, choices=sorted(WORKLOADS))
    ap.add_argument("--bt", type=int, default=0, help="force b_T (0 = planner)")
    ap.add_argument("--vec", type=int, default=0)
    ap.add_argument("--h", type=int, default=0)
    ap.add_argument("--nthr", type=int, default=0, help="threads per block of the kernel layout (0 = planner)")
    ap.add_argument("--bsy", type=int, default=0,
                    help="3D: loaded tile height b_S_y (32 = one block; 64 / 128 = a cluster of 2 / 4 blocks sharing y halos)")
    ap.add_argument("--direct", type=int, default=0, choices=[0, 1],
                    help="1 = partial sums OFF: the non-associative direct-gather kernels (BASELINE config 4)")
    ap.add_argument("--no-tune", action="store_true", help="planner model only (no measured top-5 pick)")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl", "lib"],
                    help="N > 1: halo exchange by peer stores from the sweep kernels (fused, NEXT N1), NCCL "
                         "send/recv from Python (nccl) or the library's own NCCL communicator (lib, an5d_set_comm)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="single GPU: time CUDA-graph replays of the captured T-step run (one graph per buffer parity)")
    ap.add_argument("--ref-step-seconds", type=float, default=3.0)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--T", type=int, default=0, help="override the time-step count")
    ap.add_argument("--suite", default="", help="comma list of workload names (or 'all2d', 'all3d', 'all', 'config4' = box2d2r partial sums on+off) "
                    "to run back to back at the planner's config; one JSON line each (not a driver line)")
    ap.add_argument("--bt-sweep", default="", help="with --suite: comma list of b_T values to force in turn")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.suite:
        return run_suite(args)
    return run_an5d(args)


def run_suite(args):
    """BASELINE configs 2-3: every Table-2 stencil (fp32 and fp64) at full size, one line each."""
    sel = []
    for tok in args.suite.split(","):
        if tok in ("all", "all2d"):
            sel += [w for w in WORKLOADS if w.endswith("-16384")]
        if tok in ("all", "all3d"):
            sel += [w for w in WORKLOADS if w.endswith("-512")]
        if tok in WORKLOADS:
            sel.append(tok)
        if tok == "config4":   # BASELINE config 4: box2d2r fp32, partial sums on vs off
            sel += ["box2d2r-f32-16384", "box2d2r-f32-16384@direct"]
    seen = set()
    sel = [w for w in sel if not (w in seen or seen.add(w))]
    if args.direct:
        sel = [w if "@" in w else w + "@direct" for w in sel]
    bts = [int(b) for b in args.bt_sweep.split(",") if b] or [args.bt]
    for w in sel:
        for bt in bts:
            a = argparse.Namespace(**vars(args))
            a.workload, a.bt, a.no_cpu_baseline, a.no_e2e = w.split("@")[0], bt, True, True
            if w.endswith("@direct"):
                a.direct = 1
            try:
                run_an5d(a)
            except Exception as e:  # report and continue (e.g. no instance for a forced b_T)
                print(json.dumps({"workload": w, "bT": bt, "error": str(e)[:300]}), flush=True)
    return 0


def run_an5d(args):
    import numpy as np
    import torch

    import inputs
    import paper_2001_01473_b200 as an5d
    from paper_2001_01473_b200 import perf

    ws, rank, local = _dist()
    if args.gpus > 1 or ws > 1:
        from paper_2001_01473_b200 import slab
        return slab.bench_main(args, WORKLOADS)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    name, dtype_name, n, T = WORKLOADS[args.workload]
    if args.T:
        T = args.T
    dtype = getattr(torch, dtype_name)
    nf = 1
    if name in inputs.SYSTEMS:   # multi-field system (NEXT N4): every field advanced by one kernel
        ndim, rad, shape, nf, tab = inputs.system_problem(name)
        div = 1.0
        ext = (n + 2 * rad,) * ndim
        st = an5d.System(ndim, rad, shape, tab, dtype)
        a = an5d.empty_fields(nf, ext, rad, dtype, dev)
        b = an5d.empty_fields(nf, ext, rad, dtype, dev)
        for f in range(nf):
            fill_uniform(a[f], inputs.DEFAULT_SEED + 0x1000 * f, ext)
    else:
        ndim, rad, shape, tab, div = inputs.benchmark_problem(name)
        ext = (n + 2 * rad,) * ndim
        st = an5d.Stencil(ndim, rad, shape, tab, div, dtype)
        a = an5d.empty_grid(ext, rad, dtype, dev)
        b = an5d.empty_grid(ext, rad, dtype, dev)
        fill_uniform(a, inputs.DEFAULT_SEED, ext)
    hint = {"bT": args.bt, "vec": args.vec, "h": args.h, "direct": args.direct, "n_thr": args.nthr}
    if getattr(args, "bsy", 0):
        hint["bS"] = [args.bsy, 0]
    # planner: the model's top 5 (b_T, vec) candidates run once each, fastest kept;
    # untimed, before the warm-up
    if args.no_tune:
        cfg = st.plan_config(ext, T, hint)
    else:
        cfg = st.tune(a, b, T, hint, top_k=5)
        cfg.pop("seconds_per_cell_step", None)
    geom = st.describe(ext, cfg)
    b.copy_(a)
    stream = torch.cuda.current_stream(dev)
    bufs = [a, b]

    def step(i):
        src, dst = bufs[i % 2], bufs[(i + 1) % 2]
        st.run(src, dst, T, cfg)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    launches_per_step = st.last_launch_count()
    if args.graph:
        # the whole T-step run (ring copy + every sweep) captured once per buffer parity as a CUDA
        # graph after the eager warm-up (run tables and occupancy are cached by then), replayed
        graphs = []
        for par in (0, 1):
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph):
                st.run(bufs[par], bufs[1 - par], T, cfg)
            graphs.append(gph)
        torch.cuda.synchronize()

        def step(i):
            graphs[i % 2].replay()

        for i in range(2):
            step(args.warmup + i)
        torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    cells = float(n) ** ndim * nf   # systems: cells of every field
    gcells = cells * T / (ms * 1e-3) / 1e9
    F = perf.flops_per_cell(ndim, rad, shape, div != 1.0, nf)
    peaks = _peaks()
    elem = 4 if dtype == torch.float32 else 8
    clock_mhz = peaks.get("sm_max_mhz") or 1965.0
    fp_peak = perf.fp_peak_flops(elem, 148, clock_mhz)
    nb = ndim - 1
    # 2D units are runs of stream blocks that pay the stream overlap once per run:
    # the effective stream-block length is the tile-rows per unit
    h_eff = geom["n_tiles"][0] * n / max(1, geom["n_units"]) if ndim == 2 else geom["h"]
    roof = perf.roofline(ndim=ndim, rad=rad, shape=shape, has_div=div != 1.0, dtype_bytes=elem, bT=cfg["bT"],
                         tile_loaded=geom["bS_loaded"][:nb], tile_compute=geom["compute"][:nb], h=h_eff,
                         hbm_gbs=peaks["hbm_gbs"], fp_peak=fp_peak, nf=nf)

    # ---- dominant kernel: one full-degree N.5D sweep (one persistent launch), timed per launch
    # with CUDA events on the launching stream, same grid and configuration as the step.
    n_sweep = max(5, min(50, args.steps * 5))
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(n_sweep + 1)]
    st.copy_ring(a, b)
    torch.cuda.synchronize()
    sev[0].record(stream)
    for i in range(n_sweep):
        st.sweep(bufs[i % 2], bufs[(i + 1) % 2], cfg["bT"], cfg)
        sev[i + 1].record(stream)
    torch.cuda.synchronize()
    sweep_ms = [sev[i].elapsed_time(sev[i + 1]) for i in range(n_sweep)]
    sweep_avg = statistics.mean(sweep_ms)
    alg_bytes = roof["alg_bytes_per_cell_step"] * cfg["bT"] * cells
    alg_flops = roof["alg_flops_per_cell_step"] * cfg["bT"] * cells
    sweep_cells_s = cells * cfg["bT"] / (sweep_avg * 1e-3)
    if roof["bound"] == "hbm":
        achieved = alg_bytes / (sweep_avg * 1e-3) / 1e9
        rl = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
              "frac": round(achieved / peaks["hbm_gbs"], 4)}
    else:
        achieved = alg_flops / (sweep_avg * 1e-3) / 1e12
        rl = {"bound": "alu", "achieved": round(achieved, 2), "peak": round(fp_peak / 1e12, 2), "unit": "TFLOP/s",
              "frac": round(achieved * 1e12 / fp_peak, 4)}
    tr = _traffic(args.workload, cfg)
    rl["traffic"] = tr["traffic_bytes"] if tr else None
    if tr:
        rl["traffic_source"] = tr["source"]
    rl["kernel"] = (f"an5d_sweep{ndim}d<{dtype_name},R={rad},bT={cfg['bT']},vec={cfg['vec']}"
                    f"{',direct' if cfg.get('direct') else ''}>")
    rl["sweep_ms"] = round(sweep_avg, 4)
    rl["sweep_share_of_step"] = round(sweep_avg * len(an5d.schedule(T, cfg["bT"])[0]) / ms, 4)
    rl["alg_bytes_per_launch"] = round(alg_bytes)
    rl["alg_flops_per_launch"] = round(alg_flops)
    rl["peak_source"] = (f"hbm: MEASURED_PEAKS.json hbm_gbs ({peaks['source']}); alu: CUDA-core FMA peak "
                         f"148 SM x {128 if elem == 4 else 64} FMA/clk x 2 FLOP x {clock_mhz:.0f} MHz "
                         f"(MEASURED_PEAKS sm_max_mhz; tensor cores unused: not a contraction)")
    rl["roof_gcells"] = round(roof["roof_cells_s"] / 1e9, 2)
    rl["roof_bound"] = roof["bound"]
    rl["frac_of_roof"] = round(sweep_cells_s / roof["roof_cells_s"], 4)
    rl["ideal_gcells"] = round(roof["ideal_cells_s"] / 1e9, 2)
    rl["ideal_frac"] = round(sweep_cells_s / roof["ideal_cells_s"], 4)
    rl["step_frac_of_roof"] = round(gcells * 1e9 / roof["roof_cells_s"], 4)
    rl["R_read"] = round(roof["R_read"], 4)
    rl["R_comp"] = round(roof["R_comp"], 4)
    rl["R_read_kernel"] = round(roof["R_read_kernel"], 4)

    # ---- end to end through the public API with host buffers (pinned), copies inside the region.
    # Every step copies its input grid host->device, runs T steps (an5d_run) and reads the result
    # back.  Steps are pipelined over two device buffer pairs on three streams (H2D of step i+1 and
    # D2H of step i-1 overlap the sweeps of step i; PCIe is full duplex) when the grids are small
    # enough to double-buffer; otherwise serial on one stream.
    e2e = None
    if not args.no_e2e and nf == 1:
        stor = a.untyped_storage()
        nbytes = stor.nbytes()
        k_e2e = max(2, min(args.steps, 5))
        pipelined = nbytes <= (4 << 30)
        nbuf = 2 if pipelined else 1
        host_in = [torch.empty(nbytes // elem, dtype=dtype, pin_memory=True) for _ in range(nbuf)]
        # (pinned explicitly: empty_like would return pageable memory, ~6 GB/s instead of ~50)
        host_out = [torch.empty(nbytes // elem, dtype=dtype, pin_memory=True) for _ in range(nbuf)]
        flat = lambda t: torch.empty(0, dtype=dtype, device=dev).set_(t.untyped_storage())
        for h in host_in:
            h.copy_(flat(a).cpu())
        bufs = [(a, b)] + ([(an5d.empty_grid(ext, rad, dtype, dev), an5d.empty_grid(ext, rad, dtype, dev))]
                           if pipelined else [])
        s_in = torch.cuda.Stream(dev) if pipelined else stream
        s_out = torch.cuda.Stream(dev) if pipelined else stream
        ev_comp = [torch.cuda.Event() for _ in range(nbuf)]
        ev_in = [torch.cuda.Event() for _ in range(nbuf)]
        ev_out = [torch.cuda.Event() for _ in range(nbuf)]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s_in.wait_event(e0)
        s_out.wait_event(e0)
        for i in range(k_e2e):
            j = i % nbuf
            ga, gb = bufs[j]
            if i >= nbuf:
                s_in.wait_event(ev_comp[j])       # step i-2's sweeps no longer read buffer ga
            with torch.cuda.stream(s_in):
                flat(ga).copy_(host_in[j], non_blocking=True)
            ev_in[j].record(s_in)
            stream.wait_event(ev_in[j])
            if i >= nbuf:
                stream.wait_event(ev_out[j])      # step i-2's result has been read back from gb
            st.run(ga, gb, T, cfg)
            ev_comp[j].record(stream)
            s_out.wait_event(ev_comp[j])
            with torch.cuda.stream(s_out):
                host_out[j].copy_(flat(gb), non_blocking=True)
            ev_out[j].record(s_out)
        for j in range(nbuf):
            stream.wait_event(ev_out[j])
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / k_e2e
        e2e = {"value": round(cells * T / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GCells/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": round(e2e_ms, 3),
               "steps": k_e2e, "pipelined": pipelined}
        del bufs

    cpu = None
    if not args.no_cpu_baseline and nf == 1:
        fill_uniform(a, inputs.DEFAULT_SEED, ext)
        host_grid = a.cpu().numpy()
        cpu = cpu_oracle_rate(name, dtype_name, n, host_grid, budget_s=args.cpu_budget)

    clocks = clk.summary()
    line = {
        "metric": f"GCells/s ({name} {dtype_name} {n}^{ndim}, T={T})", "value": round(gcells, 3),
        "unit": "GCells/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if dtype == torch.float32 else "f64", "data": "synthetic",
        "config": {"workload": args.workload, "stencil": name, "grid": list(ext), "n_fields": nf, "T": T, "bT": cfg["bT"],
                   "vec": cfg["vec"], "h": cfg["h"], "n_thr": cfg["n_thr"], "partial_sums": "off" if cfg.get("direct") else "on",
                   "planner": "model" if args.no_tune else "model top-5, measured pick (P:784-793)",
                   "bS": geom["bS"][:nb], "bS_loaded": geom["bS_loaded"][:nb],
                   "parallelism": "1 GPU", "l2": f"inputs larger than L2 ({a.numel() * a.element_size() / 2**30:.2f} GiB per grid buffer > 126 MB)",
                   "regs_per_thread": geom["regs_per_thread"],
                   "launch": "cuda_graph" if args.graph else "stream"},
        "gflops": round(gcells * F, 2),
        "roofline": rl,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"], "reasons": clocks["reasons"],
                   "samples": clocks["samples"]},
        "paper_v100": {"star2d1r_f32_gcells": 626, "source": "PAPER.md Table 5 P:871 (5,631 GFLOP/s / 9), V100"},
    }
    if cpu:
        cpu.pop("seconds", None)
        cpu.pop("T_sample", None)
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
