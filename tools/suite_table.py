"""Print a compact table of bench --suite JSON lines (optionally next to an older suite file)."""
import json
import sys


def load(f):
    out = {}
    for l in open(f):
        try:
            d = json.loads(l)
        except Exception:
            continue
        if "config" not in d:
            continue
        out[(d["config"]["workload"], d["config"]["bT"], d["config"].get("direct", 0))] = d
    return out


new = load(sys.argv[1])
old = load(sys.argv[2]) if len(sys.argv) > 2 else {}
oldw = {k[0]: v for k, v in old.items()}
for k, d in new.items():
    r = d.get("roofline", {})
    o = oldw.get(k[0])
    extra = f"  old {o['value']:8.1f} ({d['value'] / o['value']:.2f}x)" if o else ""
    print(f"{k[0]:22s} bT={k[1]} vec={d['config']['vec']} h={d['config']['h']:5d} {d['value']:8.1f} GC/s "
          f"frac={r.get('frac')} {r.get('bound')} regs={d['config'].get('regs_per_thread')}{extra}")
