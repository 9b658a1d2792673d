"""Stall samples of an ncu report's SASS source page, by opcode and by cause
(usage: python tools/sass_stalls.py report.ncu-rep)."""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
si = h.index("Source")
st = h.index("Warp Stall Sampling (All Samples)")
causes = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[st]) for r in data if r[st].isdigit()) or 1
byop, bycause = collections.Counter(), collections.Counter()
for r in data:
    if not r[st].isdigit():
        continue
    toks = r[si].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    byop[op.split(".")[0]] += int(r[st])
    for c in causes:
        v = r[h.index(c)]
        if v.isdigit():
            bycause[c] += int(v)
print("stall samples", tot)
for k, v in byop.most_common(14):
    print(f"  {k:10s} {100 * v / tot:5.1f}%")
for k, v in bycause.most_common(10):
    print(f"  {k:22s} {100 * v / tot:5.1f}%")
