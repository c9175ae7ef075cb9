"""Instructions per source line of an ncu capture, normalised per walk step
(executed warp instructions / (tiles x steps)), with the top SASS opcodes of
each line.  Usage: python scripts/ncu_perline.py rep.ncu-rep warp_steps [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, steps = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, fname = None, None
ex, src, ops = collections.Counter(), {}, collections.defaultdict(collections.Counter)
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    k = (fname, int(r[0]))
    src[k] = r[1].strip()[:64]
    try:
        n = int(r[hdr["Instructions Executed"]] or 0)
    except ValueError:
        n = 0
    ex[k] += n
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3] if len(r) > 3 else "")
    if m and n:
        ops[k][m.group(2)] += n
tot = sum(ex.values())
print(f"total {tot} = {tot / steps:.1f} per warp-step")
for k, v in ex.most_common(top):
    t = ", ".join(f"{o} {c / steps:.1f}" for o, c in ops[k].most_common(3))
    print(f"{k[0]}:{k[1]:4d} {v / steps:6.1f}/step  [{t}]  {src[k]}")
