"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

usage: python tools/launch_shares.py launches.csv [out.txt]
Groups launches by kernel name (template arguments kept), prints count, total ms and share of the
total device time of every launch in the list (cold-cache, serialised: compare shares, not times).
"""
import csv
import sys
from collections import defaultdict


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[r[13]]
        name = r[4][:110]
        tot[name] += float(r[14].replace(",", "")) * scale
        cnt[name] += 1
    all_ms = sum(tot.values())
    lines = [f"{len(rows)} launches, {all_ms:.1f} ms device time (ncu, serialised, cold cache)"]
    for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"{100 * ms / all_ms:6.2f} %  {cnt[name]:5d} x  {ms:9.2f} ms  {name}")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
