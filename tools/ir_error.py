"""Coarse-solve accuracy of the refinement variants at the BASELINE configs (development tool):
relative difference of A0^{-1} c and of M^{-1} x against a solve with 3 full refinement steps,
for (refine_steps, strip_refine) in {(0,0), (0,1) default, (1,0), (1,1)}."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

VARIANTS = [(0, 0), (0, 1), (1, 0), (1, 1)]
for name, (n, k, problem, p) in {"cfg2": (257, 50.0, "MP2", 8), "cfg3": (513, 100.0, "MP1", 16),
                                 "cfg4": (1025, 200.0, "MP2", 32), "cfg5": (2049, 300.0, "MP2", 64)}.items():
    grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = hb.assemble(grid, k, problem)
    dec = hb.extend(hb.partition(grid, p), 2)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(prob.A.N) + (1j * rng.standard_normal(prob.A.N) if problem == "MP2" else 0)
    ref = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, refine_steps=3, strip_refine=1)
    c = ref.restrict(x)
    y3, z3 = ref.coarse_solve(c), ref(x)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    out = []
    for ir, sr in VARIANTS:
        M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, refine_steps=ir, strip_refine=sr)
        out.append("IR%d/S%d coarse %.2e M %.2e" % (ir, sr, rel(M.coarse_solve(c), y3), rel(M(x), z3)))
        del M
    print(name, " | ".join(out), flush=True)
