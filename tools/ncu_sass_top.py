"""Top SASS instructions by warp-stall samples in an ncu report (with the two dominant reasons)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
idx = {k: i for i, k in enumerate(h)}
k = "Warp Stall Sampling (All Samples)"
rows = [x for x in r[2:] if len(x) == len(h)]
f = lambda v: float(v) if v not in ("", "-") else 0.0
tot = sum(f(x[idx[k]]) for x in rows) or 1.0
cols = [c for c in h if c.startswith("stall_")]
for i in sorted(range(len(rows)), key=lambda i: -f(rows[i][idx[k]]))[:n]:
    x = rows[i]
    top = sorted(((f(x[idx[c]]), c) for c in cols), reverse=True)[:2]
    print(f"{100 * f(x[idx[k]]) / tot:5.1f}% [{i:5d}] {x[1].strip()[:60]:60s} {top}")
