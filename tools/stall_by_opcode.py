"""Aggregate ncu source-page (SASS) stall samples by opcode for one kernel.

ncu -i rep --page source --csv --print-source sass > src.csv
python tools/stall_by_opcode.py src.csv [kernel-index]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
end = starts[k + 1] if k + 1 < len(starts) else len(rows)
print(rows[starts[k]][1][:100])
blk = rows[starts[k] + 1:end]
hdr = blk[0]
col = {h: i for i, h in enumerate(hdr)}
reasons = ["stall_dispatch", "stall_math", "stall_wait", "stall_not_selected", "stall_selected",
           "stall_short_sb", "stall_long_sb", "stall_branch_resolving", "stall_no_inst", "stall_mio"]
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in blk[1:]:
    if len(r) < len(hdr):
        continue
    op = r[col["Source"]].strip()
    op = op.split()[0] if op else "?"
    if op.startswith("@"):
        op = r[col["Source"]].strip().split()[1]
    op = op.split(".")[0]
    n = int(r[col["Instructions Executed"]] or 0)
    agg[op]["inst"] += n
    for s in reasons + ["Warp Stall Sampling (All Samples)"]:
        v = int(float(r[col[s]] or 0))
        agg[op][s] += v
        tot[s] += v
total_samples = tot["Warp Stall Sampling (All Samples)"]
print(f"total stall samples {total_samples}")
print(f"{'op':10s} {'inst':>12s} {'samples%':>8s} " + " ".join(f"{s[6:14]:>8s}" for s in reasons))
for op, c in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:18]:
    print(f"{op:10s} {c['inst']:12d} {100 * c['Warp Stall Sampling (All Samples)'] / total_samples:8.1f} " +
          " ".join(f"{100 * c[s] / total_samples:8.1f}" for s in reasons))
