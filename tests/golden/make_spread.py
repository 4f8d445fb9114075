"""Spread of the UNMODIFIED reference's GMRES count under choices its own contract allows (build container only).

The reference's iteration count on the near-resonant BASELINE configs (cfg3: 100, cfg4a: 373)
depends on rounding-level details of its own preconditioner.  This script re-runs the reference
(same objects, same inputs, same GmresConfig) varying only what the reference's specification
leaves open:

* the SuperLU fill-reducing column ordering.  SPEC.md:77 ("LU with partial pivoting on a
  fill-reducing ordering (nested-dissection-style or minimum-degree)") does not fix it;
  ``linalg.factorize`` (linalg.py:64-87) calls ``splu(A)`` with scipy's default (COLAMD).  The
  variants pass ``permc_spec`` = MMD_AT_PLUS_A / MMD_ATA (minimum degree) through to that call,
  for the coarse and the local factorizations alike.
* the order of the subdomains in the Decomposition.  SPEC ("order-independent to 1e-13") and
  pkg/tests/test_schwarz.py:153-167 permute ``index_sets``/``weights`` with
  ``dataclasses.replace`` exactly like this; the one-level sum then accumulates in another order.

Nothing else is touched: ``helmdd.linalg.splu`` is the only name rebound (to scipy's own splu
with a fixed ``permc_spec``), and the permuted Decomposition is built with dataclasses.replace.

``--coarse`` adds variants with a MORE ACCURATE coarse solve, to show where the count of an
accurate preconditioner lands (``schwarz.coarse_correct`` rebound, everything else the reference's):
``ir1``/``ir2`` = the reference's SuperLU solve plus 1/2 iterative-refinement steps with its own A0;
``dst`` = the exact fast-sine-transform diagonalisation of the Dirichlet A0 (DESIGN.md §3 K5, the
device algorithm, in numpy GEMMs; eigenvalue sums in long double); ``dst+fdm`` additionally
replaces the p^2 SuperLU local solves by the fast diagonalisation of every subdomain matrix
(DESIGN.md §3 K4, the device algorithm in numpy, ``_local_sum`` rebound).  With both the
device's algorithms inside the reference's own GMRES loop, the count shows what the device
path should give if it is correct.

Output: tests/golden/<case>_spread.json -- one record per variant (ordering, permutation seed,
iterations, converged, final residual, sampled solution norm difference against the default run).

Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_spread.py cfg3 [--orders ...] [--perms ...]
       (one variant per process: --one ORDER SEED writes a single record to stdout)
"""

from __future__ import annotations

import argparse
import functools
import json
import os
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import CASES, GMRES_RTOL, SUBSAMPLE  # noqa: E402

CAPS = {"cfg3": 200, "cfg4a": 420}


def dst_coarse_correct(name):
    """R0^T A0^{-1} R0 r with A0^{-1} by the DST-I diagonalisation (MP-1 only; fdm_setup.coarse_fast)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2408_03571_b200 import fdm_setup as F
    from paper_2408_03571_b200.discretization import Grid

    n, k = CASES[name][0], CASES[name][1]
    T0, M0, _, _, _ = F.coarse_pencil(Grid(n, "dirichlet"), k)
    m = len(T0)
    lamT, lamM = F._transform_eigs(T0.real, False), F._transform_eigs(M0.real, False)
    ld = np.longdouble
    lT, lM = lamT.astype(ld), lamM.astype(ld)
    den = (lT[:, None] * lM[None, :] + lM[:, None] * lT[None, :] - ld(k) ** 2 * np.outer(lM, lM)).astype(np.float64)
    i = np.arange(m)
    Q = np.sin(np.pi * np.outer(i + 1, i + 1) / (m + 1))
    Qi = (2.0 / (m + 1)) * Q.T

    def cc(cs, r):
        C = (cs.r0 @ r).reshape(m, m)
        return cs.r0.T @ (Q @ ((Qi @ C @ Qi.T) / den) @ Q.T).ravel()

    return cc


def fdm_local_sum(name, dec_ref):
    """SchwarzPreconditioner._local_sum (schwarz.py:64-74) with A_i^{-1} by fast diagonalisation
    (V_y (x) V_x) diag(1/(lam_y + lam_x - k^2)) (V_y (x) V_x)^T, per box, in numpy."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    import paper_2408_03571_b200 as hb
    from paper_2408_03571_b200 import fdm_setup as F

    n, k, problem, p, m = CASES[name][:5]
    g = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    d = hb.extend(hb.partition(g, p), m)
    lc = F.local_classes(g, k, d.boxes)
    mult = d.multiplicity_1d
    nu = g.unknowns_per_dim
    den = {}

    def local_sum(self, x, out, weighted):
        assert not self.weights_before_solve
        X, O = x.reshape(nu, nu), out.reshape(nu, nu)
        for ay in range(p):
            for ax in range(p):
                ys, yl, xs, xl = lc.box_start[ay], lc.box_len[ay], lc.box_start[ax], lc.box_len[ax]
                cy, cx = lc.box_class[ay], lc.box_class[ax]
                if (cy, cx) not in den:
                    den[(cy, cx)] = lc.lam[cy][:, None] + lc.lam[cx][None, :] - k**2
                Vy, Vx = lc.V[cy], lc.V[cx]
                Y = Vy @ ((Vy.T @ X[ys:ys + yl, xs:xs + xl] @ Vx) / den[(cy, cx)]) @ Vx.T
                if weighted:
                    Y = Y / np.outer(mult[ys:ys + yl], mult[xs:xs + xl])
                O[ys:ys + yl, xs:xs + xl] += Y

    return local_sum


def run_one(name: str, order: str, perm_seed: int, coarse: str = "superlu") -> dict:
    from dataclasses import replace

    import scipy.sparse.linalg as spla

    import helmdd as H
    import helmdd.linalg as L

    if order != "COLAMD":
        L.splu = functools.partial(spla.splu, permc_spec=order)  # linalg.py:79 calls splu(A)
    n, k, problem, p, m, ratio, rhs_kind, _ = CASES[name]
    t0 = time.time()
    grid = H.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = H.assemble(grid, k, problem)
    dec = H.extend(H.partition(grid, p), m)
    if perm_seed >= 0:  # pkg/tests/test_schwarz.py:153-167
        perm = np.random.default_rng(perm_seed).permutation(dec.num_subdomains)
        dec = replace(dec, index_sets=[dec.index_sets[i] for i in perm], weights=[dec.weights[i] for i in perm])
    cs = H.galerkin(H.build_hocs(grid, ratio), prob.A)
    if coarse.startswith("ir"):
        import helmdd.schwarz as S

        steps = int(coarse[2:])

        def refined(cs_, r):  # coarse.py:170-174 plus `steps` refinement steps with the same factor
            c = cs_.r0 @ r
            y = L.solve(cs_.a0_factorization, c)
            for _ in range(steps):
                y = y + L.solve(cs_.a0_factorization, c - cs_.a0 @ y)
            return cs_.r0.T @ y

        S.coarse_correct = refined
    elif coarse.startswith("dst"):
        import helmdd.schwarz as S

        S.coarse_correct = dst_coarse_correct(name)
        if coarse == "dst+fdm":
            S.SchwarzPreconditioner._local_sum = fdm_local_sum(name, dec)
    M = H.SchwarzPreconditioner("SHS2", prob.A, dec, cs)
    setup = time.time() - t0
    rep = H.gmres(prob.A, M, prob.f, H.GmresConfig(rtol=GMRES_RTOL, max_iter=CAPS[name], side="right"))
    return dict(case=name, ordering=order, perm_seed=perm_seed, coarse=coarse, iterations=int(rep.iterations),
                converged=bool(rep.converged), final_residual=float(rep.final_residual),
                coarse_fill=int(cs.a0_factorization.fill_nnz), setup_s=round(setup, 1),
                wall_s=round(rep.wall_seconds, 1), x_sample=[[float(v.real), float(v.imag)] for v in rep.x[::SUBSAMPLE * 97]],
                history_tail=[float(h) for h in rep.residual_history[-4:]])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--orders", default="COLAMD,MMD_AT_PLUS_A,MMD_ATA")
    ap.add_argument("--perms", default="-1,0,1,2")
    ap.add_argument("--coarse", default="superlu", help="comma list of superlu, ir1, ir2, dst, dst+fdm")
    ap.add_argument("--jobs", type=int, default=4)
    ap.add_argument("--one", nargs=3, metavar=("ORDER", "SEED", "COARSE"))
    a = ap.parse_args()
    if a.one:
        print(json.dumps(run_one(a.case, a.one[0], int(a.one[1]), a.one[2])), flush=True)
        return
    variants = [(o, int(s), c) for c in a.coarse.split(",") for o in a.orders.split(",") for s in a.perms.split(",")]
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1")
    out_path = os.path.join(HERE, f"{a.case}_spread.json")
    results = []
    if os.path.exists(out_path):
        with open(out_path) as f:
            results = json.load(f)["runs"]
    done = {(r["ordering"], r["perm_seed"], r.get("coarse", "superlu")) for r in results}
    todo = [v for v in variants if v not in done]
    running = []
    while todo or running:
        while todo and len(running) < a.jobs:
            o, s, c = todo.pop(0)
            pr = subprocess.Popen([sys.executable, __file__, a.case, "--one", o, str(s), c], env=env,
                                  stdout=subprocess.PIPE, text=True)
            running.append(pr)
        time.sleep(2)
        for pr in list(running):
            if pr.poll() is not None:
                running.remove(pr)
                line = pr.stdout.read().strip().splitlines()
                if pr.returncode == 0 and line:
                    rec = json.loads(line[-1])
                    results.append(rec)
                    print(json.dumps({k: rec[k] for k in ("ordering", "perm_seed", "coarse", "iterations", "converged")}), flush=True)
                    with open(out_path, "w") as f:
                        json.dump(dict(case=a.case, note=__doc__.split("\n\n")[0], runs=results), f, indent=1)


if __name__ == "__main__":
    main()
