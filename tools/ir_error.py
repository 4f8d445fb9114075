"""Coarse-solve accuracy without / with iterative refinement at the BASELINE configs (development tool):
relative difference of A0^{-1} c computed with refine_steps 0 and 1 against refine_steps 3."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

for name, (n, k, problem, p) in {"cfg2": (257, 50.0, "MP2", 8), "cfg3": (513, 100.0, "MP1", 16),
                                 "cfg4": (1025, 200.0, "MP2", 32), "cfg5": (2049, 300.0, "MP2", 64)}.items():
    grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = hb.assemble(grid, k, problem)
    dec = hb.extend(hb.partition(grid, p), 2)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(prob.A.N) + (1j * rng.standard_normal(prob.A.N) if problem == "MP2" else 0)
    Ms = {ir: hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, refine_steps=ir) for ir in (0, 1, 3)}
    c = Ms[0].restrict(x)
    ys = {ir: Ms[ir].coarse_solve(c) for ir in Ms}
    zs = {ir: Ms[ir](x) for ir in Ms}
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    print(name, "coarse IR0 %.2e IR1 %.2e" % (rel(ys[0], ys[3]), rel(ys[1], ys[3])),
          "| M IR0 %.2e IR1 %.2e" % (rel(zs[0], zs[3]), rel(zs[1], zs[3])), flush=True)
