"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
a markdown table: per kernel, launches, mean/total time, share of the listed
launches after the setup kernels.  Usage:
    python scripts/summarize_launches.py gpurun_out/r1_launches.csv > profiles/x.md"""
import csv
import re
import sys
from collections import OrderedDict

SETUP = ("coords_kernel", "qdata_kernel", "rhs_kernel", "l2e_kernel", "geo_kernel")


def short(name):
    m = re.match(r"(?:void )?([\w:<>,\s]+?)\(", name)
    n = (m.group(1) if m else name).replace("hofem::<unnamed>::", "").replace("hofem::", "")
    return n[:90]


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r["Metric Unit"], 1)
        rows.append((short(r["Kernel Name"]), r["Grid Size"], r["Block Size"], ns))
    agg = OrderedDict()
    for n, g, b, ns in rows:
        a = agg.setdefault(n, [0, 0.0, g, b])
        a[0] += 1
        a[1] += ns
    steady = sum(a[1] for n, a in agg.items() if not n.startswith(SETUP))
    print(f"source: `{path}` ({len(rows)} launches)\n")
    print("| kernel | grid | block | launches | mean (us) | total (ms) | share of non-setup |")
    print("|---|---|---|---|---|---|---|")
    for n, (c, t, g, b) in agg.items():
        sh = "setup" if n.startswith(SETUP) else f"{100 * t / steady:.1f}%"
        print(f"| `{n}` | {g} | {b} | {c} | {t / c / 1e3:.1f} | {t / 1e6:.3f} | {sh} |")


if __name__ == "__main__":
    main(sys.argv[1])
