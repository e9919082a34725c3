"""Write profiles/ncu_traffic.json from ncu --set full captures (run here).

    python tools/ncu_traffic_update.py <workload> <tag> <report.ncu-rep> [...]

Per kernel base name (stageA_kernel, stageC_kernel, joint_kernel, ...):
dram__bytes_read.sum + dram__bytes_write.sum summed over the captured launches
of one step (stage C is one launch per decode-pool class), and the issue-slot
utilisation / SIMT efficiency weighted by launch duration.  bench.py reads
`bytes` as roofline.traffic, `issue_active` as the measured issue-slot
fraction and `warp_instr_per_request` (smsp__inst_executed.sum ÷ the simulated
requests the kernel processes per step, SURVEY §8(d) event roofline) of the
dominant kernel.  Works on --set full reports and on the short metric list

    ncu --metrics {METRICS} ...
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
     "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
     "inst": "smsp__inst_executed.sum"}
METRICS = ",".join(M.values())
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
            if m not in hdr:
                d[k] = float("nan")
                continue
            i = hdr.index(m)
            v = float(vals[i].replace(",", "") or "nan")
            d[k] = v * SCALE.get(units[i], 1.0)
        name = vals[hdr.index("Kernel Name")]
        d["name"] = name.split("(")[0].split("<")[0].split("::")[-1].replace("void ", "").strip()
        d["kw"] = None
        if d["name"] == "stageC_kernel" and "<" in name:     # <CTX, IDX, KW, BL>: decode-pool class
            d["kw"] = int(name.split("<")[1].split(">")[0].split(",")[2])
        yield d


def requests_per_kernel(wl):
    """Simulated requests each replay kernel processes in one step of `wl`."""
    sys.path.insert(0, ROOT)
    import oracle
    from bench import build_workload
    from workloads import get_config
    cfg = get_config(wl)
    role, cap, pols, traces, qps, _ = build_workload(cfg, 0, oracle.enumerate_pool_uniform)
    r_sum = sum(int(t["s_unit"].size) for t in traces)
    st = [c for c in range(role.shape[0]) if pols[c]["kind"] == 0]
    groups = {tuple(int(v) for v in cap[c][role[c] == 0]) for c in st}
    Q, C = len(qps), role.shape[0]
    if cfg["n_gpus"] <= 8:
        # stage C launches one kernel per decode-pool class (padsim.cu plan_factorized:
        # five classes KW = 1, 2, 4, 5, 7 for ≥ 400 k static replays, else KW = 2, 4, 7)
        fine = len(st) * Q * len(traces) >= 400000
        kw = {}
        for c in st:
            y = int((role[c] == 1).sum())
            k = (1 if y <= 1 else 2 if y <= 2 else 4 if y <= 4 else 5 if y <= 5 else 7) if fine else \
                (2 if y <= 2 else 4 if y <= 4 else 7)
            kw[k] = kw.get(k, 0) + Q * r_sum
        return {"stageA_kernel": len(groups) * Q * r_sum, "stageC_kernel": len(st) * Q * r_sum,
                "joint_kernel": (C - len(st)) * Q * r_sum, "_stageC_kw": kw}
    # N > 8: static candidates on the wide-node factorized path, dynamic ones on the joint kernel
    return {"stageA_wide_kernel": len(groups) * Q * r_sum, "stageC_wide_kernel": len(st) * Q * r_sum,
            "joint_kernel": (C - len(st)) * Q * r_sum}


def main():
    wl, tag, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    req = requests_per_kernel(wl)
    agg = defaultdict(lambda: defaultdict(float))
    missing = defaultdict(int)
    for p in reps:
        for d in rows(p):
            if any(d[k] != d[k] for k in ("dur", "iss")):     # NaN: ncu did not collect
                missing[d["name"]] += 1
                continue
            a = agg[d["name"]]
            a["launches"] += 1
            if d["kw"] is not None:
                a["req"] += req.get("_stageC_kw", {}).get(d["kw"], 0)
            a["read"] += d["rd"] if d["rd"] == d["rd"] else 0.0
            a["write"] += d["wr"] if d["wr"] == d["wr"] else 0.0
            a["dur"] += d["dur"]
            a["inst"] += d["inst"] if d["inst"] == d["inst"] else 0.0
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
                "warp_instr": a["inst"],
                # per request of the launches collected (stage C: their decode-pool classes)
                "warp_instr_per_request": (a["inst"] / (a["req"] or req[n])) if req.get(n) and a["inst"] else None,
                "requests": a["req"] or req.get(n),
                "launches_not_collected": missing.get(n, 0)}
    json.dump(data, open(OUT, "w"), indent=1)
    print(json.dumps(w, indent=1))


if __name__ == "__main__":
    main()
