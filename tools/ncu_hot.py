"""Per-source-line hot spots of an ncu --set full report (--import-source on).

    python tools/ncu_hot.py <report.ncu-rep> [top]

Aggregates warp-stall samples of the SASS instructions under each CUDA source
line (ncu --page source --print-source cuda,sass) and prints the top lines with
their dominant stall reasons.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
files = {}
cur = None
agg = defaultdict(lambda: defaultdict(float))
src = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or cur is None or len(r) < len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    key = (cur, ln)
    src[key] = r[1].strip()
    for k, v in d.items():
        if k in ("Warp Stall Sampling (All Samples)", "Instructions Executed") or k.startswith("stall_"):
            try:
                agg[key][k] += float(v)
            except ValueError:
                pass
tot = sum(a["Warp Stall Sampling (All Samples)"] for a in agg.values()) or 1.0
lines = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]
print(f"{'file:line':28s} {'samp%':>6s} {'inst(M)':>8s}  top stalls | source")
for key, a in lines:
    s = a["Warp Stall Sampling (All Samples)"]
    st = sorted(((v, k) for k, v in a.items() if k.startswith("stall_") and "Not Issued" not in k), reverse=True)[:3]
    sts = " ".join(f"{k[6:]}:{100 * v / max(s, 1):.0f}%" for v, k in st if v > 0)
    print(f"{key[0] + ':' + str(key[1]):28s} {100 * s / tot:6.2f} {a['Instructions Executed'] / 1e6:8.1f}  {sts} | {src[key][:90]}")
