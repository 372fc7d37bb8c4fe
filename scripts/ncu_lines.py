"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.
ncu's SASS page (addresses + samples) is mapped to lines through nvdisasm -g
of the locally built cubin of the same source (offsets from function start).
usage: python scripts/ncu_lines.py report.ncu-rep cubin mangled_substring [P1]"""
import csv
import io
import re
import subprocess
import sys


def sass_samples(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ia, isamp, isrc = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    res = []
    for r in rows[2:]:
        try:
            res.append((int(r[ia], 16), int(r[isamp]), r[isrc].strip()))
        except (ValueError, IndexError):
            pass
    base = res[0][0]
    return [(a - base, s, src) for a, s, src in res]


def line_map(cubin, fn_sub):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    parts = re.split(r"\n\s*\.text\.(\S+):", txt)
    for i in range(1, len(parts), 2):
        if fn_sub in parts[i]:
            m, line, fname = {}, None, None
            for l in parts[i + 1].split("\n"):
                g = re.search(r'File "([^"]+)", line (\d+)', l)
                if g:
                    fname, line = g.group(1).split("/")[-1], int(g.group(2))
                    continue
                g = re.search(r"/\*([0-9a-f]{4,})\*/", l)
                if g:
                    m[int(g.group(1), 16)] = (fname, line)
            return m
    raise SystemExit("function not found")


def main(rep, cubin, fn_sub):
    samples = sass_samples(rep)
    lm = line_map(cubin, fn_sub)
    agg, tot, miss = {}, 0, 0
    for off, s, src in samples:
        tot += s
        key = lm.get(off)
        if key is None:
            miss += s
            continue
        agg[key] = agg.get(key, 0) + s
    print(f"total samples {tot}, unmapped {miss}")
    for (f, l), s in sorted(agg.items(), key=lambda kv: -kv[1])[:45]:
        print(f"{s:7d} {100 * s / tot:5.1f}%  {f}:{l}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
