"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel count, total and share."""
import collections
import csv
import sys


def load(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    return [r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]


def short(name):
    name = name.split("(")[0]
    return name.replace("void ", "")[:70]


if __name__ == "__main__":
    rows = load(sys.argv[1])
    skip = sys.argv[2] if len(sys.argv) > 2 else "at::"
    agg = collections.OrderedDict()
    for r in rows:
        k = short(r["Kernel Name"]) + " " + r["Grid Size"] + "x" + r["Block Size"]
        if skip and skip in r["Kernel Name"]:
            continue
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + float(r["Metric Value"]) / 1e3)
    tot = sum(t for _, t in agg.values())
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{t:10.1f} us {100 * t / tot:5.1f}%  x{c:<4d} {k}")
    print(f"{tot:10.1f} us total")
