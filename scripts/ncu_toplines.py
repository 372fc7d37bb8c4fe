"""Top CUDA source lines of one ncu report by warp-stall samples (cuda,sass view;
needs -lineinfo and --import-source).  usage: python scripts/ncu_toplines.py report.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[2]
idx = {h: i for i, h in reversed(list(enumerate(hdr)))}
S = "Warp Stall Sampling (All Samples)"
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
per = collections.defaultdict(collections.Counter)
text = {}
ln = None
for r in rows[3:]:
    if r and r[0].strip().isdigit():
        ln = int(r[0])
        text[ln] = r[1] if len(r) > 1 else ""
        continue
    if ln is None or len(r) < 4 or not r[2].startswith("0x"):
        continue
    for k in reasons + [S]:
        try:
            per[ln][k] += float(r[idx[k]] or 0)
        except (ValueError, KeyError):
            pass
tot = sum(c[S] for c in per.values()) or 1
for ln, c in sorted(per.items(), key=lambda kv: -kv[1][S])[:n]:
    top = sorted(((c[k], k) for k in reasons), reverse=True)[:3]
    why = " ".join(f"{k.replace('stall_', '')}={100 * v / tot:.1f}" for v, k in top if v)
    print(f"{100 * c[S] / tot:5.1f}% L{ln:<5d} {why:45s} {text.get(ln, '').strip()[:70]}")
