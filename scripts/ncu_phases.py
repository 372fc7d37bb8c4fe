"""Summarize an ncu report: per-barrier-phase stall samples and smem wavefronts."""
import csv
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kfilter:
    cmd += ["-k", kfilter]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
ix = hdr.index("Warp Stall Sampling (All Samples)")
iw = hdr.index("L1 Wavefronts Shared")
ie = hdr.index("L1 Wavefronts Shared Excessive")
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
bars = [i for i, r in enumerate(data) if "BAR.SYNC" in r[1]]
bounds = [0] + bars + [len(data)]
tot_all = sum(int(r[ix] or 0) for r in data)
print("kernel:", rows[0][1][:100], "samples", tot_all)
for a, b in zip(bounds[:-1], bounds[1:]):
    tot = sum(int(data[i][ix] or 0) for i in range(a, b))
    w = sum(int(data[i][iw] or 0) for i in range(a, b))
    e = sum(int(data[i][ie] or 0) for i in range(a, b))
    reasons = {s: sum(int(data[i][hdr.index(s)] or 0) for i in range(a, b)) for s in st}
    top = sorted(reasons.items(), key=lambda kv: -kv[1])[:4]
    print(f"{a:5d}-{b:5d} {100*tot/max(tot_all,1):5.1f}% smem wf {w:10d} excess {e:9d}",
          " ".join(f"{k[6:]}={v}" for k, v in top))
