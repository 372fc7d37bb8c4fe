"""Per-stage stall breakdown from an ncu report's source page (cuda,sass view;
needs -lineinfo and --import-source).  Lines are grouped by the
'// ---- <stage>' markers of the kernel source as it was when profiled.
usage: python scripts/ncu_stage_lines.py report.ncu-rep source.cuh [first_line last_line]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, src = sys.argv[1], sys.argv[2]
# helper functions attributed as their own stage (brick epilogue), found by name
EXTRA = []
_src = open(src).read().split("\n")
for _i, _l in enumerate(_src, 1):
    if re.match(r"__device__ __forceinline__ void (epi_segment|epi_dispatch|brick_epilogue)\(", _l):
        _j = _i
        while _j < len(_src) and _src[_j - 1] != "}":
            _j += 1
        EXTRA.append((_i, _j))
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10**9)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[2]
idx = {}
for i, h in enumerate(hdr):
    idx.setdefault(h, i)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
marks = []
for i, l in enumerate(open(src), 1):
    m = re.search(r"// ---- (\S+?)[:.]", l)
    if m and lo <= i <= hi:
        marks.append((i, m.group(1)))
# other code (helpers inlined from elsewhere) keeps the stage of the caller: attribute by the
# most recent kernel-body line seen in SASS order
S = "Warp Stall Sampling (All Samples)"
agg = collections.defaultdict(collections.Counter)
tot = collections.Counter()
cur = "pre"


def stage(ln):
    st = None
    for m, n in marks:
        if ln >= m:
            st = n
    return st


# SASS rows in address order; a helper line (inlined from outside the kernel
# body) takes the stage of the last kernel-body line before it
sass = []
ln = None
for r in rows[3:]:
    if r[0].strip().isdigit():
        ln = int(r[0])
        continue
    if ln is None or len(r) < 4 or not r[2].startswith("0x"):
        continue
    sass.append((int(r[2], 16), ln, r))
sass.sort()
st = "pre"
for _, ln, r in sass:
    if lo <= ln <= hi:
        st = stage(ln) or st
    elif any(a <= ln <= b for a, b in EXTRA):
        st = "epilogue"
    for k in reasons + ["Instructions Executed", S]:
        try:
            v = float(r[idx[k]] or 0)
        except ValueError:
            v = 0.0
        agg[st][k] += v
        tot[k] += v
print(f"{'stage':8s} samp% inst%  top stall reasons (% of all samples)")
for st, c in sorted(agg.items(), key=lambda kv: -kv[1][S]):
    top = sorted(((c[k], k) for k in reasons), reverse=True)[:6]
    print(f"{str(st):8s} {100 * c[S] / tot[S]:5.1f} {100 * c['Instructions Executed'] / tot['Instructions Executed']:5.1f}  "
          + " ".join(f"{k[6:]}={100 * v / tot[S]:.1f}" for v, k in top))
