"""Static SASS instruction mix per kernel of libhelmb200.so (cuobjdump -sass): the FP64 tensor-pipe
(DMMA), FP64 CUDA-core, async-copy (LDGSTS / UTMALDG / UBLKCP) and memory instructions.
Usage: python tools/sass_mix.py > profiles/sass_mix_r02.txt"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2408_03571_b200", "libhelmb200.so")
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
cur, per = None, collections.defaultdict(collections.Counter)
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur:
        per[cur][m.group(2)] += 1
elf = subprocess.run(["cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout
keys = ["DMMA", "DFMA", "DADD", "DMUL", "LDGSTS", "UTMALDG", "UBLKCP", "LDG", "STG", "LDS", "STS", "SHFL", "BAR"]
names = subprocess.run(["c++filt"], input="\n".join(per), capture_output=True, text=True).stdout.splitlines()
print("# SASS instruction mix of libhelmb200.so (cuobjdump -sass; static counts per kernel)")
print("# cubin targets:", ", ".join(sorted(set(re.findall(r"sm_\d+a?", elf)))))
print(f"{'kernel':72s} " + " ".join(f"{k:>7s}" for k in keys))
tot = collections.Counter()
for (f, c), nm in sorted(zip(per.items(), names), key=lambda kv: -sum(kv[0][1].values())):
    tot.update(c)
    nm = re.sub(r"^void ", "", nm)[:72]
    print(f"{nm:72s} " + " ".join(f"{c.get(k, 0):7d}" for k in keys))
print(f"{'TOTAL':72s} " + " ".join(f"{tot.get(k, 0):7d}" for k in keys))
