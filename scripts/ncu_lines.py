"""Per-source-line summary of an ncu capture (SASS rows correlated to CUDA
lines): executed instructions, stall samples and the top stall reasons per
line.  Usage: python scripts/ncu_lines.py rep.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
ex_by, smp_by, st_by, src = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter), {}
fname = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    src[key] = r[1].strip()[:70]
    try:
        ex_by[key] += int(r[hdr["Instructions Executed"]] or 0)
        smp_by[key] += int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        for h, i in hdr.items():
            if h.startswith("stall_") and "(" not in h and r[i]:
                st_by[key][h[6:]] += int(r[i])
    except ValueError:
        pass
tot_ex, tot_s = sum(ex_by.values()), sum(smp_by.values())
print(f"executed {tot_ex} samples {tot_s}")
for key, s in smp_by.most_common(top):
    st = ", ".join(f"{k} {v * 100 // max(s, 1)}%" for k, v in st_by[key].most_common(3))
    print(f"{key[0]}:{key[1]:4d} smp {s * 100 / tot_s:5.1f}% ex {ex_by[key] * 100 / tot_ex:5.1f}%  [{st}]  {src[key]}")
