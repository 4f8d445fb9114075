"""One paper-table cell (MP-1, maximal overlap; default: Table 4, n=129, k=30, HOCS H=16h, SHS2):
device vs oracle operators and left-preconditioned GMRES.  Args: n k ratio coarse kind."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import helmdd_oracle as O
import paper_2408_03571_b200 as hb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 129
k = float(sys.argv[2]) if len(sys.argv) > 2 else 30.0
ratio = int(sys.argv[3]) if len(sys.argv) > 3 else 16
ck = sys.argv[4] if len(sys.argv) > 4 else "HOCS"
kind = sys.argv[5] if len(sys.argv) > 5 else "SHS2"
p = (n - 1) // ratio
grid = hb.Grid(n, "dirichlet")
prob = hb.assemble(grid, k, "MP1")
dec = hb.extend_max(hb.partition(grid, p))
cs = hb.galerkin((hb.build_hocs if ck == "HOCS" else hb.build_focs)(grid, ratio), prob.A)
oprob, odec, ocs, oM = O.build_shs2(n, k, "MP1", p, "max", ratio, kind=kind, coarse=ck)
x = np.random.default_rng(1).standard_normal(prob.A.N)
for rs in (0, 2, 4):
    M = hb.SchwarzPreconditioner(kind, prob.A, dec, cs, refine_steps=rs)
    c = ocs.r0 @ x
    e_c = np.linalg.norm(M.coarse_solve(c) - ocs.lu.solve(c)) / np.linalg.norm(ocs.lu.solve(c))
    e_m = np.linalg.norm(M(x) - oM(x)) / np.linalg.norm(oM(x))
    y = np.zeros_like(x)
    e_l = np.linalg.norm(M.local_sum(x) - oM.local_sum(x, y, True)) / np.linalg.norm(y)
    rep = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-7, max_iter=200, side="left"))
    print(f"refine {rs}: coarse {e_c:.2e} local {e_l:.2e} M {e_m:.2e} GMRES {rep.iterations} {rep.converged}")
    print("  hist", np.array2string(rep.residual_history[44:56], precision=3))
orep = O.gmres(oprob.A, oM, oprob.f, 1e-7, 200, "left")
print("oracle", orep.iterations, np.array2string(orep.residual_history[44:56], precision=3))
