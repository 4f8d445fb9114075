"""How accurate are the reference's own inner solves?  (build container only)

Runs the UNMODIFIED reference at a BASELINE config and measures, on the seed-1 operator vector,
the relative distance of its SuperLU local sum (schwarz.py:64-74) and coarse solve (coarse.py:174)
from the same solves with iterative refinement (same factors, residuals with the reference's own
matrices).  Writes tests/golden/<case>_accuracy.json.

Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/reference_accuracy.py cfg3
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import CASES, operator_input  # noqa: E402


def main(name):
    import helmdd as H
    from helmdd import linalg
    from helmdd.decomposition import local_matrix

    n, k, problem, p, m, ratio, _, _ = CASES[name]
    grid = H.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = H.assemble(grid, k, problem)
    dec = H.extend(H.partition(grid, p), m)
    cs = H.galerkin(H.build_hocs(grid, ratio), prob.A)
    M = H.SchwarzPreconditioner("SHS2", prob.A, dec, cs)
    N = prob.A.shape[0]
    x = operator_input(N, problem == "MP2").astype(np.result_type(prob.A.dtype, float))
    raw = np.zeros_like(x)
    M._local_sum(x, raw, weighted=True)
    ref = np.zeros_like(x)
    for i, (idx, w, F) in enumerate(zip(dec.index_sets, dec.weights, M.local_factorizations)):
        Ai = local_matrix(dec, i, prob.A).tocsr()
        y = linalg.solve(F, x[idx])
        for _ in range(2):
            y = y + linalg.solve(F, x[idx] - Ai @ y)
        ref[idx] += w * y
    c = cs.r0 @ x
    y0 = linalg.solve(cs.a0_factorization, c)
    y2 = y0
    for _ in range(3):
        y2 = y2 + linalg.solve(cs.a0_factorization, c - cs.a0 @ y2)
    out = dict(case=name, local_sum_vs_refined=float(np.linalg.norm(raw - ref) / np.linalg.norm(ref)),
               coarse_solve_vs_refined=float(np.linalg.norm(y0 - y2) / np.linalg.norm(y2)),
               note="the reference's SuperLU solves against the same solves with 2 (local) / 3 (coarse) "
                    "iterative-refinement steps on its own matrices, seed-1 operator vector")
    with open(os.path.join(HERE, name + "_accuracy.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["cfg3"]:
        main(nm)
