"""Per-opcode warp-stall samples, executed instructions and shared-memory
wavefronts of one kernel in an ncu report (source page, SASS view).
usage: sass_opcode_mix.py <report.ncu-rep>"""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h, data = rows[0], rows[1:]
iS, iSmp = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
iW, iE = h.index("L1 Wavefronts Shared"), h.index("Instructions Executed")
tot, wf, ex, n = (collections.Counter() for _ in range(4))
for r in data:
    if len(r) < len(h) or not r[iS].split():
        continue
    parts = r[iS].split()
    op = (parts[1] if parts[0].startswith("@") else parts[0]).split(".")[0]
    tot[op] += int(r[iSmp] or 0)
    wf[op] += int(float(r[iW] or 0))
    ex[op] += int(float(r[iE] or 0))
    n[op] += 1
S = sum(tot.values()) or 1
for op, v in tot.most_common(16):
    print(f"{op:8s} stall samples {100 * v / S:5.1f}%  warp instrs {ex[op]:>12d}  smem wavefronts {wf[op]:>12d}  static {n[op]}")
print("total shared-memory wavefronts", sum(wf.values()))
