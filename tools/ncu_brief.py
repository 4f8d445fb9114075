"""Brief summary of a one-kernel ncu report: SOL, occupancy, top stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(det.splitlines()))
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
keep = ["Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Block Limit Shared Mem", "Block Limit Registers", "Memory Throughput"]
print(rows[1][ix["Kernel Name"]][:80])
for r in rows[1:]:
    if r[ix["Metric Name"]] in keep:
        print(f'  {r[ix["Metric Name"]]:32s} {r[ix["Metric Value"]]:>12s} {r[ix["Metric Unit"]]}')
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hh, vv = rr[0], rr[2]
st = [(k, x) for k, x in zip(hh, vv) if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and x not in ("", "0")]
tot = sum(float(x) for _, x in st)
print("  stalls:", ", ".join(f'{k.replace("smsp__pcsamp_warps_issue_stalled_", "")} {100*float(x)/tot:.0f}%' for k, x in sorted(st, key=lambda kv: -float(kv[1]))[:6]))
for k, x in zip(hh, vv):
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"):
        print(f"  {k} {x}")
