"""Summarise an ncu --set full report (.ncu-rep) into a small JSON for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json [label]

Per kernel launch: name, duration, DRAM bytes read/write (the roofline `traffic`), DRAM
throughput %, FMA-pipe and issue utilisation, warps per SM, registers, smem, top stall reasons.
Runs here (no GPU needed): `ncu -i ... --page raw --csv`.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_per_sm",
    "launch__registers_per_thread": "regs",
    "launch__shared_mem_per_block_dynamic": "smem_dyn",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_active.avg": "sm_active_cycles",
    "smsp__inst_executed.sum": "warp_instructions",
}


def _num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return x


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:160]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = _num(r[i])
                u = units[i]
                if name in ("dram_read", "dram_write") and isinstance(v, float):
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
                    v = v * scale
                if name == "duration_ns" and isinstance(v, float):
                    v = v * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)
                d[name] = v
        stalls = {}
        for i, k in enumerate(hdr):
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                v = _num(r[i])
                if isinstance(v, float):
                    stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = v
        tot = sum(stalls.values()) or 1.0
        d["stalls_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
        if isinstance(d.get("dram_read"), float) and isinstance(d.get("dram_write"), float):
            d["traffic_bytes"] = d["dram_read"] + d["dram_write"]
        res.append(d)
    return res


if __name__ == "__main__":
    rep, dst = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else rep
    with open(dst, "w") as f:
        json.dump({"report": label, "launches": summarise(rep)}, f, indent=1)
    print(open(dst).read())
