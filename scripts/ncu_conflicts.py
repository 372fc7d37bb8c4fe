"""Attribute shared-memory bank-conflict excess wavefronts and warp-stall
samples of one kernel in an ncu report to CUDA source lines (through the
locally built cubin of the same source, nvdisasm -g).
usage: python scripts/ncu_conflicts.py report.ncu-rep cubin mangled_substring [top]"""
import csv
import io
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from ncu_lines import line_map  # noqa: E402


def main(rep, cubin, fn, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ia, iex = h.index("Address"), h.index("L1 Wavefronts Shared Excessive")
    isamp = h.index("Warp Stall Sampling (All Samples)")
    res = []
    for r in rows[2:]:
        try:
            res.append((int(r[ia], 16), float(r[iex] or 0), int(r[isamp] or 0)))
        except (ValueError, IndexError):
            pass
    base = res[0][0]
    lm = line_map(cubin, fn)
    agg, tex, ts = {}, 0.0, 0
    for a, ex, s in res:
        k = lm.get(a - base, ("?", 0))
        d = agg.setdefault(k, [0.0, 0])
        d[0] += ex
        d[1] += s
        tex += ex
        ts += s
    print(f"excess wavefronts {tex:.3g}, stall samples {ts}")
    for (f, l), (ex, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(top)]:
        print(f"{f}:{l:5d}  excess {100 * ex / max(tex, 1):5.1f}%  samples {100 * s / max(ts, 1):5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
