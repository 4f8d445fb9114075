import os, sys
os.environ["HELM_GMRES_TRACE"] = "1"
import numpy as np
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb
grid = hb.Grid(2049, "sommerfeld")
prob = hb.assemble(grid, 300.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 64), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A))
r = np.random.default_rng(0)
b = r.standard_normal(prob.A.N) + 1j * r.standard_normal(prob.A.N)
for _ in range(2):
    rep = hb.gmres(prob.A, M, b, hb.GmresConfig(rtol=1e-30, max_iter=50))
    print("run", rep.wall_seconds, file=sys.stderr, flush=True)
