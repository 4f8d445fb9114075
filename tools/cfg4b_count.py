"""Device GMRES iteration count for BASELINE config 4(b) (n=1025, k=200, seed-0 random RHS)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

grid = hb.Grid(1025, "sommerfeld")
prob = hb.assemble(grid, 200.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 32), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A))
r = np.random.default_rng(0)
b = r.standard_normal(prob.A.N) + 1j * r.standard_normal(prob.A.N)
rep = hb.gmres(prob.A, M, b, hb.GmresConfig(rtol=1e-6, max_iter=1000))
print("cfg4b", rep.iterations, rep.converged, rep.final_residual, rep.wall_seconds)
