"""Reference GMRES with ONE iterative-refinement step added to its own coarse solve (build container only).

The reference's iteration counts on the near-resonant BASELINE configs depend on the
rounding of its SuperLU coarse solve (~5e-14 relative).  This script runs the
UNMODIFIED reference objects, replacing only ``schwarz.coarse_correct`` by
``R0^T (y + A0^{-1}(R0 r - A0 y))`` with ``y = A0^{-1} R0 r`` -- the same SuperLU
factor, one refinement step -- to measure where the count of the *more accurate*
reference preconditioner lands.  Output: tests/golden/<case>_refined.json.

With ``--coarse-ir C --local-ir L`` (C refinement steps on the coarse solve, L on every
local SuperLU solve) it writes <case>_exact.json instead: the count of a reference
preconditioner accurate to ~1e-15, used where even the singly-refined count still moves.

Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_refined.py cfg3 cfg4a
       PYTHONPATH=/root/reference/pkg/src python tests/golden/make_refined.py --coarse-ir 2 --local-ir 1 cfg4a
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


def run(name, coarse_ir=1, local_ir=0):
    import helmdd as H
    import helmdd.schwarz as S
    from helmdd import linalg
    from helmdd.decomposition import local_matrix

    def refined(cs, r):
        c = cs.r0 @ r
        y = linalg.solve(cs.a0_factorization, c)
        for _ in range(coarse_ir):
            y = y + linalg.solve(cs.a0_factorization, c - cs.a0 @ y)
        return cs.r0.T @ y

    S.coarse_correct = refined
    n, k, problem, p, m, ratio, rhs_kind, _ = CASES[name]
    grid = H.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = H.assemble(grid, k, problem)
    dec = H.extend(H.partition(grid, p), m)
    cs = H.galerkin(H.build_hocs(grid, ratio), prob.A)
    M = H.SchwarzPreconditioner("SHS2", prob.A, dec, cs)
    if local_ir:
        local_A = [local_matrix(dec, i, prob.A).tocsr() for i in range(dec.num_subdomains)]

        def local_sum(x, out, weighted):  # SchwarzPreconditioner._local_sum (schwarz.py:64-74) + refinement
            for idx, w, F, Ai in zip(dec.index_sets, dec.weights, M.local_factorizations, local_A):
                xi = x[idx]
                yi = linalg.solve(F, xi)
                for _ in range(local_ir):
                    yi = yi + linalg.solve(F, xi - Ai @ yi)
                out[idx] += (w * yi) if weighted else yi

        M._local_sum = local_sum
    b = prob.f if rhs_kind == "point" else random_rhs(prob.A.shape[0])
    t0 = time.time()
    rep = H.gmres(prob.A, M, b, H.GmresConfig(rtol=GMRES_RTOL, max_iter=GMRES_CAP, side="right"))
    out = dict(case=name, refine_steps=coarse_ir, local_refine_steps=local_ir, iterations=rep.iterations, converged=bool(rep.converged),
               final_residual=rep.final_residual, wall_s=round(time.time() - t0, 1),
               history=[float(v) for v in rep.residual_history])
    tag = "_refined" if (coarse_ir, local_ir) == (1, 0) else "_exact"
    with open(os.path.join(HERE, name + tag + ".json"), "w") as f:
        json.dump(out, f)
    print(json.dumps({k: v for k, v in out.items() if k != "history"}), flush=True)


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="+")
    ap.add_argument("--coarse-ir", type=int, default=1)
    ap.add_argument("--local-ir", type=int, default=0)
    a = ap.parse_args()
    for nm in a.cases:
        run(nm, a.coarse_ir, a.local_ir)
