"""Per-CUDA-source-line summary of an ncu --set full report (shared-memory wavefronts, the
excess from bank conflicts, local-memory (spill) traffic, warp-stall samples):
    python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, cur, data = None, "", []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and len(r) == len(hdr):
        d = {}
        for k, v in zip(hdr, r):
            d.setdefault(k, v)  # the first "Source" column is the CUDA line
        d["_file"] = cur
        data.append(d)


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


def col(name):
    return sum(num(d.get(name)) for d in data)


print(f"shared wavefronts {col('L1 Wavefronts Shared'):.4g}  excessive "
      f"{col('L1 Wavefronts Shared Excessive'):.4g}  stall samples "
      f"{col('Warp Stall Sampling (All Samples)'):.4g}")
for label, k in (("shared wavefronts", "L1 Wavefronts Shared"),
                 ("excess wavefronts (bank conflicts)", "L1 Wavefronts Shared Excessive"),
                 ("local-memory (spill) L2 sectors", "L2 Theoretical Sectors Local"),
                 ("stall samples", "Warp Stall Sampling (All Samples)")):
    print("== top lines by", label)
    for d in sorted(data, key=lambda d: -num(d.get(k)))[:top]:
        v = num(d.get(k))
        if v <= 0:
            break
        print(f"{v:11.4g}  {d['_file']}:{d['Line No']:<5} {d.get('Source', '').strip()[:100]}")
