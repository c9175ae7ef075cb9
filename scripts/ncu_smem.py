"""Shared-memory wavefronts per source line of an ncu capture (SASS rows
correlated to CUDA lines): total, ideal and excessive wavefronts.
Usage: python scripts/ncu_smem.py rep.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
wf, ideal, exc, src, ops = (collections.Counter(), collections.Counter(), collections.Counter(), {},
                            collections.defaultdict(collections.Counter))
fname, hdr = None, None
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

    def num(h):
        try:
            return int(float(r[hdr[h]] or 0))
        except (ValueError, KeyError):
            return 0
    wf[key] += num("L1 Wavefronts Shared")
    ideal[key] += num("L1 Wavefronts Shared Ideal")
    exc[key] += num("L1 Wavefronts Shared Excessive")
    op = r[3].split()[0] if len(r) > 3 and r[3] else "?"
    if num("L1 Wavefronts Shared"):
        ops[key][op.split(".")[0] if not op.startswith("@") else r[3].split()[1].split(".")[0]] += 1
tw, te = sum(wf.values()), sum(exc.values())
print(f"shared wavefronts {tw}, excessive {te} ({te * 100 / max(tw, 1):.1f}%)")
for key, v in wf.most_common(top):
    print(f"{key[0]}:{key[1]:4d} wf {v * 100 / tw:5.1f}% exc {exc[key] * 100 / max(tw, 1):5.1f}% ideal {ideal[key]}  "
          f"{dict(ops[key])}  {src[key]}")
