"""Per-iteration table of the device GMRES at config 5: for each Arnoldi step j the device
times of the operator (M^-1 at batch 1 + A x) and of CGS2 (HELM_GMRES_TRACE=1 brackets them with CUDA
events; the look-ahead is off in that mode), against the HBM roofline of the step's algorithmic bytes.
Writes a text table to stdout.  Usage: python tools/gmres_per_j.py [iterations]"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r'''
import sys
sys.path.insert(0, %r)
import numpy as np
import paper_2408_03571_b200 as hb
n, k, p, iters = 2049, 300.0, 64, int(sys.argv[1])
grid = hb.Grid(n, "sommerfeld")
prob = hb.assemble(grid, k, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, p), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A))
r0 = np.random.default_rng(0)
b = r0.standard_normal(prob.A.N) + 1j * r0.standard_normal(prob.A.N)
cfg = hb.GmresConfig(rtol=1e-300, max_iter=iters)
hb.gmres(prob.A, M, b, cfg)
print("MARK", file=sys.stderr, flush=True)
rep = hb.gmres(prob.A, M, b, cfg)
print("REORTH", rep.reorth_iterations, file=sys.stderr, flush=True)
''' % ROOT


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    r = subprocess.run([sys.executable, "-c", CHILD, str(iters)], env=dict(os.environ, HELM_GMRES_TRACE="1"),
                       capture_output=True, text=True)
    err = r.stderr.split("MARK")[-1]
    rows = [(int(m.group(1)), float(m.group(2)), float(m.group(3)))
            for m in re.finditer(r"gmres it (\d+) wall [\d.]+ ms op ([\d.]+) cgs2 ([\d.]+)", err)]
    try:
        bw = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        bw = 6536.4
    N = 2049 * 2049
    Ns = N * 16
    print(f"# device GMRES, config 5 operator, seed-0 random complex right-hand side, {iters} iterations, rtol 1e-300")
    print(f"# op = M^-1 (batch 1) + A x; CGS2 = the basis sweeps of step j; roofline = (3(j+1)+4) N s / {bw:.0f} GB/s "
          "(SURVEY §8(d), three sweeps; the device skips the third where gmres.py:117-120 does)")
    print(f"{'j':>3s} {'op ms':>8s} {'cgs2 ms':>8s} {'cgs2 roof ms':>12s} {'cgs2 frac':>9s}")
    for j, op, cg in rows:
        roof = (3 * (j + 1) + 4) * Ns / (bw * 1e9) * 1e3
        print(f"{j:3d} {op:8.3f} {cg:8.3f} {roof:12.3f} {roof / cg if cg else 0:9.2f}")
    if rows:
        print(f"# mean op {sum(r[1] for r in rows) / len(rows):.3f} ms, mean CGS2 {sum(r[2] for r in rows) / len(rows):.3f} ms")
    m = re.search(r"REORTH (\d+)", err)
    if m:
        print(f"# second orthogonalisation pass ran in {m.group(1)} of {len(rows)} iterations")


if __name__ == "__main__":
    main()
