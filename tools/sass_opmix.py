"""Per-opcode instruction mix and warp-stall attribution from an ncu source-page CSV.

usage: python tools/sass_opmix.py SOURCE.csv OUT.json
SOURCE.csv = `ncu -i REPORT.ncu-rep --page source --csv --print-source sass` (runs without a GPU).
Per opcode: warp instructions executed, stall samples, and the top stall reasons on it.
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
kernel, hdr, data = rows[0][1], rows[1], rows[2:]
i_s, i_e = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = {h: hdr.index(h) for h in hdr if h.startswith("stall_") and "Not Issued" not in h}
exe, smp, why = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
for r in data:
    toks = [t for t in r[1].strip().split() if not t.startswith("@")]
    if not toks or not r[i_e].isdigit():
        continue
    op = toks[0].split(".")[0]
    exe[op] += int(r[i_e])
    smp[op] += int(r[i_s]) if r[i_s].isdigit() else 0
    for c, i in stall_cols.items():
        if r[i].isdigit():
            why[op][c] += int(r[i])
tot_e, tot_s = sum(exe.values()), sum(smp.values())
total_why = collections.Counter()
for c in why.values():
    total_why.update(c)
out = {"kernel": kernel, "warp_instructions": tot_e, "stall_samples": tot_s,
       "stall_reasons": {k: round(v / tot_s, 3) for k, v in total_why.most_common(10)},
       "opcodes": [{"op": op, "executed": n, "frac_executed": round(n / tot_e, 4),
                    "stall_frac": round(smp[op] / tot_s, 4),
                    "top_stalls": {k: v for k, v in why[op].most_common(3)}}
                   for op, n in exe.most_common(30)]}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps({k: out[k] for k in ("warp_instructions", "stall_samples", "stall_reasons")}))
