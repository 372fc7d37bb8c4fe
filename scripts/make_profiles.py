"""Write profiles/<tag>_* summaries from a gpurun_out/<tag>/ capture directory:
launch list (csv + markdown share table), ncu --set full summaries (markdown +
raw csv export) and profiles/traffic.json (DRAM bytes per fused launch, read by
bench.py's roofline).  usage: python scripts/make_profiles.py r1c"""
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def main(tag, dst=None):
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = dst or os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    if os.path.exists(os.path.join(src, "launches.csv")):
        shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, f"{tag}_launches.csv"))
        with open(os.path.join(dst, f"{tag}_launches.md"), "w") as f:
            f.write(run([sys.executable, os.path.join(ROOT, "scripts", "summarize_launches.py"),
                         os.path.join(src, "launches.csv")]))
    tpath = os.path.join(dst, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for rep in sorted(glob.glob(os.path.join(src, "*.ncu-rep"))):
        name = os.path.splitext(os.path.basename(rep))[0]
        with open(os.path.join(dst, f"{tag}_{name}.md"), "w") as f:
            f.write(run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep]))
        raw = run(["ncu", "-i", rep, "--page", "raw", "--csv"])
        with open(os.path.join(dst, f"{tag}_{name}_raw.csv"), "w") as f:
            f.write(raw)
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            kn = r[h.index("Kernel Name")]
            if "fused_elem" not in kn and "fused_column" not in kn:
                continue
            def val(k):
                i = h.index(k)
                v = float(r[i].replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1)
            b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            import re
            mm = re.match(r"simt_p(\d+)(?:_(\d+)x(\d+)x(\d+))?$", name)
            if mm:
                p = int(mm.group(1))
                if mm.group(2):
                    key = f"bp3_p{p}_{mm.group(2)}x{mm.group(3)}x{mm.group(4)}"
                else:
                    n = int(round(311.0 / p))
                    key = f"bp3_p{p}_{n}x{n}x{n}"
                traffic[key] = {"dram_bytes": b, "kernel": kn[:80],
                                "source": f"profiles/{tag}_{name}_raw.csv"}
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1)
    print("wrote", sorted(os.listdir(dst)))


if __name__ == "__main__":
    # usage: make_profiles.py <tag> [--out DIR]  (DIR: e.g. gpurun_out/<tag>/profiles on
    # the GPU box, so only the small summaries travel back)
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    if out:
        os.makedirs(out, exist_ok=True)
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            shutil.copy(tp, os.path.join(out, "traffic.json"))
    main(sys.argv[1], out)
