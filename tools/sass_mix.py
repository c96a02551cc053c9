"""Instruction mix of the hot loop of an ncu --set full report (source page, SASS).

usage: python tools/sass_mix.py REPORT.ncu-rep [frac]
Instructions executed at least `frac` (default 0.5) times the most executed one form the hot
loop; prints per-opcode shares of executed instructions and of warp-stall samples.
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(rep, frac=0.5):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    isrc, iss, iex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    mx = max(float(r[iex] or 0) for r in data)
    tot = sum(float(r[iss] or 0) for r in data)
    hot = [r for r in data if float(r[iex] or 0) >= float(frac) * mx]
    c, s = Counter(), Counter()
    for r in hot:
        t = r[isrc].strip().split()
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        c[op] += float(r[iex])
        s[op] += float(r[iss])
    T = sum(c.values())
    print(f"hot loop: {len(hot)} instructions, {sum(s.values()) / tot * 100:.1f} % of stall samples")
    for op, v in c.most_common(30):
        print(f"{op:10s} {v / T * 100:6.2f} % instr  {s[op] / tot * 100:6.2f} % samples")


if __name__ == "__main__":
    main(*sys.argv[1:])
