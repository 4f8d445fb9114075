"""Diagnose a GMRES iteration-count mismatch: device GMRES vs the oracle's MGS GMRES driving the
GPU preconditioner vs the oracle end to end, plus operator parity on the same config (development tool)."""
import sys, time
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import helmdd_oracle as O
import paper_2408_03571_b200 as hb
from common import load_golden, operator_input, rel

CFG = {"cfg2": (257, 50.0, "MP2", 8), "cfg3": (513, 100.0, "MP1", 16), "cfg4a": (1025, 200.0, "MP2", 32)}
name = sys.argv[1]
n, k, problem, p = CFG[name]
g = load_golden(name)
grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
prob = hb.assemble(grid, k, problem)
dec = hb.extend(hb.partition(grid, p), 2)
M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, hb.galerkin(hb.build_hocs(grid, 2), prob.A))
oprob, odec, ocs, oM = O.build_shs2(n, k, problem, p, 2)
x = operator_input(prob.A.N, problem == "MP2")
y0 = np.zeros(prob.A.N, dtype=np.result_type(x.dtype, oprob.A.dtype))
print("A x", rel(prob.A @ x, oprob.A @ x))
print("R0 x", rel(M.restrict(x), ocs.r0 @ x))
c = ocs.r0 @ x
print("coarse", rel(M.coarse_solve(c), ocs.lu.solve(c)))
print("R0^T", rel(M.prolong(c), ocs.r0.T @ c))
print("local", rel(M.local_sum(x), oM.local_sum(x.astype(y0.dtype), y0.copy(), True)))
print("M", rel(M(x), oM(x)))
rd = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-6, max_iter=1000))
print("device gmres", rd.iterations, flush=True)
t = time.time()
ro = O.gmres(oprob.A, lambda v: M(v), oprob.f, 1e-6, 1000)
print("oracle gmres + GPU M", ro.iterations, f"{time.time()-t:.1f}s", flush=True)
hg = g["gmres_history"]
for j in range(0, min(len(hg), len(rd.residual_history), len(ro.residual_history)), 5):
    print(j, f"{hg[j]:.4e} {ro.residual_history[j]:.4e} {rd.residual_history[j]:.4e}")
