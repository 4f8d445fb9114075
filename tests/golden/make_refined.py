"""Reference GMRES with ONE iterative-refinement step added to its own coarse solve (build container only).

The reference's iteration counts on the near-resonant BASELINE configs depend on the
rounding of its SuperLU coarse solve (~5e-14 relative).  This script runs the
UNMODIFIED reference objects, replacing only ``schwarz.coarse_correct`` by
``R0^T (y + A0^{-1}(R0 r - A0 y))`` with ``y = A0^{-1} R0 r`` -- the same SuperLU
factor, one refinement step -- to measure where the count of the *more accurate*
reference preconditioner lands.  Output: tests/golden/<case>_refined.json.

Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_refined.py cfg3 cfg4a
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import CASES, GMRES_CAP, GMRES_RTOL, random_rhs  # noqa: E402


def run(name):
    import helmdd as H
    import helmdd.schwarz as S
    from helmdd import linalg

    def refined(cs, r):
        c = cs.r0 @ r
        y = linalg.solve(cs.a0_factorization, c)
        y = y + linalg.solve(cs.a0_factorization, c - cs.a0 @ y)
        return cs.r0.T @ y

    S.coarse_correct = refined
    n, k, problem, p, m, ratio, rhs_kind, _ = CASES[name]
    grid = H.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = H.assemble(grid, k, problem)
    dec = H.extend(H.partition(grid, p), m)
    cs = H.galerkin(H.build_hocs(grid, ratio), prob.A)
    M = H.SchwarzPreconditioner("SHS2", prob.A, dec, cs)
    b = prob.f if rhs_kind == "point" else random_rhs(prob.A.shape[0])
    t0 = time.time()
    rep = H.gmres(prob.A, M, b, H.GmresConfig(rtol=GMRES_RTOL, max_iter=GMRES_CAP, side="right"))
    out = dict(case=name, refine_steps=1, iterations=rep.iterations, converged=bool(rep.converged),
               final_residual=rep.final_residual, wall_s=round(time.time() - t0, 1),
               history=[float(v) for v in rep.residual_history])
    with open(os.path.join(HERE, name + "_refined.json"), "w") as f:
        json.dump(out, f)
    print(json.dumps({k: v for k, v in out.items() if k != "history"}), flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        run(nm)
