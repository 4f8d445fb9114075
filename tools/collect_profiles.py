"""Copy one evidence run (tools/gpu_evidence.sh, TAG) from gpurun_out/ into profiles/ as text summaries:
launch lists with per-kernel time share and DRAM bytes (batch 32 / 1), the top-kernel ncu brief, bench
lines, the GPU test log and smoke.  Usage: python tools/collect_profiles.py r02_v1"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1]


def launches(path, title, bw=6536.4):
    with open(path) as f:
        rows = list(csv.DictReader([l for l in f if l.startswith('"')]))
    agg = collections.OrderedDict()
    for r in rows:
        if "helm::" not in r["Kernel Name"]:
            continue
        k = r["Kernel Name"].split("(")[0].replace("void ", "")[:60]
        key = (k, r["ID"])
        d = agg.setdefault(k, {"n": set(), "t": 0.0, "rd": 0.0, "wr": 0.0})
        d["n"].add(r["ID"])
        v = float(r["Metric Value"])
        name, unit = r["Metric Name"], r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
        if name == "gpu__time_duration.sum":
            d["t"] += v * scale.get(unit, 1)
        elif name == "dram__bytes_read.sum":
            d["rd"] += v * scale.get(unit, 1)
        elif name == "dram__bytes_write.sum":
            d["wr"] += v * scale.get(unit, 1)
    tot = sum(d["t"] for d in agg.values())
    out = [f"# {title}", "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
           "--clock-control none (cold cache, serialised); two applies; HBM peak 6536 GB/s (MEASURED_PEAKS.json)",
           f"{'kernel':60s} {'launches':>8s} {'us/launch':>10s} {'share':>6s} {'MB/launch':>10s} {'GB/s':>8s} {'of peak':>7s}"]
    for k, d in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        n = len(d["n"])
        us = d["t"] / n / 1e3
        mb = (d["rd"] + d["wr"]) / n / 1e6
        gbs = mb / 1e3 / (us / 1e6) if us else 0.0
        out.append(f"{k:60s} {n:8d} {us:10.1f} {100 * d['t'] / tot:5.1f}% {mb:10.1f} {gbs:8.1f} {gbs / bw:7.2f}")
    out.append(f"total {tot / 1e3 / 2:.1f} us per apply (serialised, cold)")
    return "\n".join(out) + "\n"


def write(name, text):
    with open(os.path.join(P, name), "w") as f:
        f.write(text)
    print("wrote", name)


if os.path.exists(os.path.join(G, f"launches_M_{tag}.csv")):
    write(f"launches_M_b32_{tag}.txt", launches(os.path.join(G, f"launches_M_{tag}.csv"),
                                                "one SHS2 M^-1 at config 5, batch 32"))
if os.path.exists(os.path.join(G, f"launches_M_b1_{tag}.csv")):
    write(f"launches_M_b1_{tag}.txt", launches(os.path.join(G, f"launches_M_b1_{tag}.csv"),
                                               "one SHS2 M^-1 at config 5, batch 1 (the GMRES operator)"))
rep = os.path.join(G, f"top_kernel_{tag}.ncu-rep")
if os.path.exists(rep):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_brief.py"), rep], capture_output=True,
                         text=True).stdout
    write(f"top_kernel_local_fdm_dmma_{tag}.txt", txt)
for src, dst in ((f"bench_{tag}.log", f"bench_{tag}.jsonl"), (f"bench_ref_{tag}.log", f"bench_ref_{tag}.jsonl")):
    p = os.path.join(G, src)
    if os.path.exists(p):
        lines = [l for l in open(p) if l.startswith("{")]
        if lines:
            write(dst, lines[-1])
for src in (f"pytest_gpu_{tag}.txt", f"smoke_{tag}.log"):
    p = os.path.join(G, src)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(P, src))
        print("copied", src)
