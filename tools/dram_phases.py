"""Per-phase DRAM bytes of one batch-32 SHS2 apply from a launch-list summary (profiles/launches_M_b32_<tag>.txt,
written by collect_profiles.py from the ncu CSV): writes profiles/dram_traffic_<round>.json, which bench.py
reads for roofline.traffic.  Usage: python tools/dram_phases.py r02_v5 r02"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rnd = sys.argv[1], sys.argv[2]
PHASE = {
    "restrict_sweep": "R0 x", "prolong_deflate": "R0^T c + deflate",
    "local_": "local sum", "combine_kernel": "local sum",
    "xform_": "coarse solve", "band_solve": "coarse solve", "band_tma": "coarse solve", "strip_": "coarse solve",
}
tot = {}
src = os.path.join(ROOT, "profiles", f"launches_M_b32_{tag}.txt")
for line in open(src):
    if not line.startswith("helm::") or "band_seg_setup" in line:
        continue  # the one-time segmented-solve setup is not part of an apply
    f = line.split()
    name = f[0][len("helm::"):]
    # columns from the right: launches us/launch share MB/launch GB/s of-peak (kernel names may hold spaces)
    launches, mb = int(f[-6]), float(f[-3])
    for key, ph in PHASE.items():
        if name.startswith(key):
            tot[ph] = tot.get(ph, 0.0) + launches / 2 * mb * 1e6  # the list covers two applies
            break
    else:
        raise SystemExit(f"unmapped kernel {name}")
out = {k: int(v) for k, v in tot.items()}
out["_note"] = (f"DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per batch-32 SHS2 apply at n=2049, summed over "
                f"the phase's kernels (one-time band_seg setup excluded); ncu --metrics ... --clock-control none on "
                f"tools/profile_ops.py --only M^-1 (profiles/launches_M_b32_{tag}.txt)")
with open(os.path.join(ROOT, "profiles", f"dram_traffic_{rnd}.json"), "w") as fo:
    json.dump(out, fo, indent=1)
print(json.dumps(out, indent=1))
