"""Per-stage warp-stall breakdown of a fused kernel from an ncu report: SASS
rows mapped to source lines through the local cubin (see ncu_lines.py), lines
grouped by the '// ---- <stage>' markers of fused_impl.cuh.
usage: python scripts/ncu_stages.py report cubin mangled_substring"""
import csv
import io
import re
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import ncu_lines as N  # noqa: E402

REASONS = ["stall_wait", "stall_short_sb", "stall_long_sb", "stall_barrier", "stall_math",
           "stall_mio", "stall_lg", "stall_selected", "stall_not_selected", "stall_branch_resolving",
           "stall_dispatch", "stall_no_inst"]


def stages(src_path):
    marks = []
    for i, l in enumerate(open(src_path), 1):
        m = re.search(r"// ---- (S\w+):", l)
        if m:
            marks.append((i, m.group(1)))
    return marks


def main(rep, cubin, fn_sub):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ia = h.index("Address")
    idx = {r: h.index(r) for r in REASONS if r in h}
    itot = h.index("Warp Stall Sampling (All Samples)")
    iinst = h.index("Instructions Executed")
    recs = []
    for r in rows[2:]:
        try:
            recs.append((int(r[ia], 16), r))
        except ValueError:
            pass
    base = recs[0][0]
    lm = N.line_map(cubin, fn_sub)
    src = sys.argv[4] if len(sys.argv) > 4 else "paper_2402_15940_b200/csrc/fused_impl.cuh"
    marks = stages(src)
    # kernel body range: stage markers after the kernel's first marker
    agg = {}
    for a, r in recs:
        f, l = lm.get(a - base, ("?", 0))
        name = "other"
        if f == "fused_impl.cuh":
            cand = [m for m in marks if m[0] <= l]
            name = cand[-1][1] if cand else f"line<{marks[0][0]}"
            if l < 400:
                name = "helpers(<400: lattice/epilogue/brick)"
            elif not cand or l < marks[0][0]:
                name = "kernel preamble / ld_row"
        d = agg.setdefault(name, {"tot": 0, "inst": 0, **{k: 0 for k in idx}})
        d["tot"] += int(r[itot] or 0)
        d["inst"] += int(r[iinst] or 0)
        for k, i in idx.items():
            d[k] += int(r[i] or 0)
    tot = sum(d["tot"] for d in agg.values())
    print(f"{'stage':40s} {'samples%':>8s} {'inst%':>6s} " + " ".join(f"{k[6:]:>8s}" for k in idx))
    itot_all = sum(d["inst"] for d in agg.values())
    for name, d in sorted(agg.items(), key=lambda kv: -kv[1]["tot"]):
        print(f"{name[:40]:40s} {100 * d['tot'] / tot:8.1f} {100 * d['inst'] / itot_all:6.1f} " +
              " ".join(f"{100 * d[k] / tot:8.1f}" for k in idx))


if __name__ == "__main__":
    main(*sys.argv[1:4])
