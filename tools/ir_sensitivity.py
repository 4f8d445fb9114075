"""GMRES count vs coarse refinement steps on a BASELINE config (development tool)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

CFG = {"cfg2": (257, 50.0, "MP2", 8), "cfg3": (513, 100.0, "MP1", 16), "cfg4a": (1025, 200.0, "MP2", 32)}
name = sys.argv[1]
n, k, problem, p = CFG[name]
grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
prob = hb.assemble(grid, k, problem)
dec = hb.extend(hb.partition(grid, p), 2)
cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
xs = {}
for ir in (0, 1, 2, 3):
    M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, refine_steps=ir)
    rep = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-6, max_iter=1000))
    xs[ir] = rep.x
    print(name, "refine", ir, "iterations", rep.iterations, "true", rep.final_residual,
          "x vs IR0 %.2e" % (np.linalg.norm(rep.x - xs[0]) / np.linalg.norm(xs[0])), flush=True)
