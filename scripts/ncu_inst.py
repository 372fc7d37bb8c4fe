"""Per-barrier-phase executed instruction mix from an ncu report (SASS source page)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
ie = hdr.index("Instructions Executed")
bars = [i for i, r in enumerate(data) if "BAR.SYNC" in r[1]]
bounds = [0] + bars + [len(data)]
tot = sum(int(r[ie] or 0) for r in data)
print("total warp-instructions", tot)
for a, b in zip(bounds[:-1], bounds[1:]):
    c = collections.Counter()
    n = 0
    for i in range(a, b):
        k = int(data[i][ie] or 0)
        op = data[i][1].split()[0] if data[i][1].split() else "?"
        if op.startswith("@"):
            op = data[i][1].split()[1]
        c[op.split(".")[0]] += k
        n += k
    top = ", ".join(f"{k}={v/1e6:.1f}M" for k, v in c.most_common(7))
    print(f"{a:5d}-{b:5d} {n/1e6:8.1f}M ({100*n/tot:4.1f}%)  {top}")
