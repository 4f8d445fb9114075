import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb
grid = hb.Grid(2049, "sommerfeld")
prob = hb.assemble(grid, 300.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 64), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A))
r = np.random.default_rng(0)
b = r.standard_normal(prob.A.N) + 1j * r.standard_normal(prob.A.N)
rep = hb.gmres(prob.A, M, b, hb.GmresConfig(rtol=1e-30, max_iter=40))
np.set_printoptions(precision=3, linewidth=150)
print(rep.residual_history)
print(rep.iterations, rep.converged, rep.breakdown, rep.final_residual)
rep = hb.gmres(prob.A, M, b, hb.GmresConfig(rtol=1e-6, max_iter=400))
print(rep.iterations, rep.converged, rep.breakdown, rep.final_residual)
print(rep.residual_history[::20])
