"""Print section/metric/value rows of an ncu report's details page for kernels matching a regex."""
import csv, re, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
want = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, si, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
seen = set()
for r in rows[1:]:
    if len(r) <= vi or not re.search(pat, r[ki]):
        continue
    key = (r[0], r[si], r[mi])
    if key in seen:
        continue
    seen.add(key)
    if want and not want.search(r[si] + " " + r[mi]):
        continue
    print(f"[{r[0]}] {r[si][:28]:28s} {r[mi][:55]:55s} {r[vi]:>14s} {r[ui]}")
