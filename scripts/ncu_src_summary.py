"""Summarise an ncu source page (SASS): instruction mix, stall reasons, top
stalled instructions.  Usage: python scripts/ncu_src_summary.py rep.ncu-rep [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
ex = idx["Instructions Executed"]
smp = idx["Warp Stall Sampling (All Samples)"]
tot_ex = sum(int(r[ex]) for r in data)
tot_s = sum(int(r[smp]) for r in data)
print(f"executed {tot_ex}  samples {tot_s}")
cols = [c for c in hdr if c.startswith("stall_") and "(" not in c]
tot = collections.Counter()
for r in data:
    for c in cols:
        tot[c] += int(r[idx[c]])
s = sum(tot.values())
print("stalls:", ", ".join(f"{c[6:]} {v / s * 100:.1f}%" for c, v in tot.most_common(9)))
byop, byop_s = collections.Counter(), collections.Counter()
for r in data:
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1])
    op = m.group(2) if m else r[1]
    byop[op] += int(r[ex])
    byop_s[op] += int(r[smp])
print("mix:", ", ".join(f"{op} {c / tot_ex * 100:.1f}%" for op, c in byop.most_common(18)))
for r in sorted(data, key=lambda r: -int(r[smp]))[:top]:
    print(r[0][-5:], f"{int(r[smp]):7d} ex{int(r[ex]):10d}", r[1][:58].strip(),
          {c[6:]: r[idx[c]] for c in cols if int(r[idx[c]]) > 0.2 * int(r[smp])})
