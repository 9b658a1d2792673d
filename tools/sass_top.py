"""Top stalled SASS instructions of an ncu report with their dominant stall cause and the
few instructions before them (usage: sass_top.py report.ncu-rep [n] [kernel index])."""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
his = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r]
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = his[which]; end = his[which + 1] if which + 1 < len(his) else len(rows)
h = rows[hi]; data = [r for r in rows[hi + 1:end] if len(r) == len(h)]
si = h.index("Source"); st = h.index("Warp Stall Sampling (All Samples)")
causes = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[st]) for r in data if r[st].isdigit()) or 1
order = sorted(range(len(data)), key=lambda i: -int(data[i][st]) if data[i][st].isdigit() else 0)[:n]
for i in sorted(order):
    r = data[i]
    cs = sorted(((int(r[h.index(c)]) if r[h.index(c)].isdigit() else 0, c) for c in causes), reverse=True)[:2]
    print(f"{i:5d} {100*int(r[st])/tot:5.2f}%  {r[si][:70]:70s} {cs[0][1]}:{cs[0][0]} {cs[1][1]}:{cs[1][0]}")
    for k in range(max(0, i - 2), i):
        print(f"        . {data[k][si][:90]}")
