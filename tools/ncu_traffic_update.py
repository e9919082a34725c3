"""Write profiles/ncu_traffic.json from ncu --set full captures (run here).

    python tools/ncu_traffic_update.py <workload> <tag> <report.ncu-rep> [...]

Per kernel base name (stageA_kernel, stageC_kernel, joint_kernel, ...):
dram__bytes_read.sum + dram__bytes_write.sum summed over the captured launches
of one step (stage C is one launch per decode-pool class), and the issue-slot
utilisation / SIMT efficiency weighted by launch duration.  bench.py reads
`bytes` as roofline.traffic and `issue_active` as the measured issue-slot
fraction of the dominant kernel.
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")
M = {"dur": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
     "iss": "sm__inst_issued.avg.pct_of_peak_sustained_active",
     "simt": "smsp__thread_inst_executed_per_inst_executed.ratio",
     "warps": "sm__warps_active.avg.pct_of_peak_sustained_active"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def rows(path):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"]).decode()
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    for vals in r[2:]:
        d = {}
        for k, m in M.items():
            i = hdr.index(m)
            v = float(vals[i].replace(",", ""))
            d[k] = v * SCALE.get(units[i], 1.0)
        name = vals[hdr.index("Kernel Name")]
        d["name"] = name.split("(")[0].split("<")[0].split("::")[-1].replace("void ", "").strip()
        yield d


def main():
    wl, tag, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    agg = defaultdict(lambda: defaultdict(float))
    missing = defaultdict(int)
    for p in reps:
        for d in rows(p):
            if any(d[k] != d[k] for k in ("rd", "wr", "iss")):     # NaN: ncu did not collect
                missing[d["name"]] += 1
                continue
            a = agg[d["name"]]
            a["launches"] += 1
            a["read"] += d["rd"]
            a["write"] += d["wr"]
            a["dur"] += d["dur"]
            for k in ("iss", "simt", "warps"):
                a[k] += d[k] * d["dur"]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["_source"] = ("ncu --set full --clock-control none captures (tools/ncu_traffic_update.py): "
                       "dram bytes summed over the launches of one step; issue-slot / SIMT / warp "
                       "occupancy duration-weighted")
    w = data.setdefault(wl, {})
    for n, a in agg.items():
        w[n] = {"bytes": a["read"] + a["write"], "read": a["read"], "write": a["write"],
                "launches": int(a["launches"]), "ncu_ms": a["dur"] * 1e3,
                "issue_active": a["iss"] / a["dur"] / 100, "simt_threads": a["simt"] / a["dur"],
                "warps_active": a["warps"] / a["dur"] / 100, "profile": tag,
                "launches_not_collected": missing.get(n, 0)}
    json.dump(data, open(OUT, "w"), indent=1)
    print(json.dumps(w, indent=1))


if __name__ == "__main__":
    main()
