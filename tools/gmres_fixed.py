"""Fixed-length GMRES run at n=2049 (rtol 1e-300, seed-0 random RHS) as in bench.py: ms per iteration
(development tool; env switches HELM_PDL / HELM_GMRES_LOOKAHEAD / HELM_GMRES_TRACE apply)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 1
grid = hb.Grid(2049, "sommerfeld")
prob = hb.assemble(grid, 300.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 64), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A), max_batch=mb)
r0 = np.random.default_rng(0)
b = r0.standard_normal(prob.A.N) + 1j * r0.standard_normal(prob.A.N)
cfg = hb.GmresConfig(rtol=1e-300, max_iter=iters)
for rep_i in range(3):
    rep = hb.gmres(prob.A, M, b, cfg)
    print(f"run {rep_i}: {rep.iterations} it, {1e3 * rep.wall_seconds / rep.iterations:.4f} ms/it", flush=True)
