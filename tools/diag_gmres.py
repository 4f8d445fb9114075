import sys, os, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import helmdd_oracle as O
import paper_2408_03571_b200 as hb
from common import load_golden
g = load_golden("cfg2")
n,k,p = 257, 50.0, 8
grid = hb.Grid(n, "sommerfeld"); prob = hb.assemble(grid, k, "MP2")
dec = hb.extend(hb.partition(grid, p), 2); cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs)
Acsr = prob.A.tocsr()
ro = O.gmres(Acsr, lambda v: M(v), prob.f, 1e-6, 100)
rd = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-6, max_iter=100))
rn = hb.gmres(prob.A, None, prob.f, hb.GmresConfig(rtol=1e-6, max_iter=30))
rno = O.gmres(Acsr, None, prob.f, 1e-6, 30)
print("oracle-gmres with GPU M:", ro.iterations, "device:", rd.iterations, "golden:", int(g["gmres_iterations"]))
hg = g["gmres_history"]
for j in range(min(len(hg), len(rd.residual_history), len(ro.residual_history))):
    print(j, hg[j], ro.residual_history[j], rd.residual_history[j])
print("unpreconditioned:", [ (a,b) for a,b in zip(rno.residual_history[:31], rn.residual_history[:31])][-3:])
