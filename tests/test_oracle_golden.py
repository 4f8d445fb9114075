"""Pin the CPU oracle (oracle/helmdd_oracle.py) against the reference's own outputs.

The fixtures in tests/golden were produced by running the unmodified reference
(tests/golden/make_golden.py).  The oracle must reproduce every operator to
1e-12 and the GMRES iteration count to +-1 (SuperLU is not bitwise
deterministic across processes, SURVEY hazard H12).
"""

import numpy as np
import pytest

import helmdd_oracle as O
from common import golden_names, load_golden, operator_input, random_rhs, reference_count, rel

VEC = golden_names(store_vectors=True)


def build(g):
    n, k, problem, p, m = int(g["n"]), float(g["k"]), str(g["problem"]), int(g["p"]), int(g["overlap_layers"])
    return O.build_shs2(n, k, problem, p, m)


@pytest.mark.parametrize("name", VEC)
def test_oracle_operators(name):
    g = load_golden(name)
    prob, dec, cs, M = build(g)
    x = operator_input(prob.A.shape[0], prob.problem == "MP2")
    c = cs.r0 @ x
    assert rel(c, g["R0x"]) <= 1e-14
    assert rel(cs.lu.solve(c), g["coarse_solve"]) <= 1e-12
    assert rel(M(x), g["M_shs2"]) <= 1e-12
    if "Ax" in g:
        assert rel(prob.A @ x, g["Ax"]) <= 1e-15
        assert rel(cs.r0.T @ c, g["R0T_c"]) <= 1e-15
        y = np.zeros(prob.A.shape[0], dtype=np.result_type(x.dtype, prob.A.dtype))
        assert rel(M.local_sum(x.astype(y.dtype), y, True), g["local_sum"]) <= 1e-12
        for kind in ("AS2", "SAS2"):
            Mk = O.OSchwarz(kind, prob.A, dec, cs)
            assert rel(Mk(x), g["M_" + kind.lower()]) <= 1e-12


@pytest.mark.parametrize("name", VEC + ["cfg3"])
def test_oracle_gmres(name):
    g = load_golden(name)
    prob, dec, cs, M = build(g)
    b = prob.f if str(g["gmres_rhs"]) == "point" else random_rhs(prob.A.shape[0])
    rep = O.gmres(prob.A, M, b, 1e-6, 1000)
    assert rep.converged == bool(g["gmres_converged"])
    assert abs(rep.iterations - int(g["gmres_iterations"])) <= 1
    assert rep.final_residual <= 1e-6
    if rep.iterations == int(g["gmres_iterations"]) and "gmres_x" in g and name not in ("cfg2",):
        assert rel(rep.x, g["gmres_x"]) <= 1e-8


def test_dense_oracle_tiny():
    """Matrix-free SHS2/AS2/SAS2 == explicit dense operator (test_schwarz.py:22-62 style), HOCS ratio 2."""
    for n, k, problem, p, m in [(9, 2.0, "MP1", 4, 2), (17, 3.0, "MP2", 2, 2), (17, 5.0, "MP2", 4, 3)]:
        prob, dec, cs, _ = O.build_shs2(n, k, problem, p, m)
        for kind in ("AS2", "SAS2", "SHS2"):
            M = O.OSchwarz(kind, prob.A, dec, cs)
            dense = O.dense_preconditioner(kind, prob.A, dec, cs)
            eye = np.eye(prob.A.shape[0], dtype=prob.A.dtype)
            got = np.column_stack([M(e) for e in eye])
            assert np.abs(got - dense).max() < 1e-11 * np.abs(dense).max()


def test_paper_known_answer_hocs_h4():
    """Paper/acceptance known answer (test_acceptance.py:37-60): MP-2, k=20,
    n=81, H_sub = H = 4h, max overlap, HOCS ratio 4, left preconditioning: SHS2 converges in 8."""
    grid = O.OGrid(81, "sommerfeld")
    prob = O.assemble(grid, 20.0, "MP2")
    dec = O.decompose(grid, 20, 2)  # extend_max: m = c // 2 = 2 for c = 4
    cs = O.coarse_space(grid, prob.A, 4)
    M = O.OSchwarz("SHS2", prob.A, dec, cs)
    rep = O.gmres(prob.A, M, prob.f, 1e-7, 100, side="left")
    assert rep.converged and rep.iterations == 8


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_oracle_refined_coarse_counts(name):
    """The reference with one refinement step on its SuperLU coarse solve (tests/golden/make_refined.py)
    and the oracle with the same step agree on the GMRES count."""
    import json
    import os

    from common import GOLDEN

    g = load_golden(name)
    with open(os.path.join(GOLDEN, name + "_refined.json")) as f:
        refined = int(json.load(f)["iterations"])
    raw = reference_count(name, g)
    prob, dec, cs, _ = build(g)
    M = O.OSchwarz("SHS2", prob.A, dec, cs, coarse_refine=1)
    rep = O.gmres(prob.A, M, prob.f, 1e-6, 1000)
    assert rep.converged and abs(rep.iterations - refined) <= 1, (rep.iterations, refined, raw)


def test_oracle_large_goldens_cfg3():
    """The oracle against the sampled config-3 goldens of the unmodified reference
    (tests/golden/make_golden_large.py): every operator <= 1e-12 on sample, norm and functional."""
    import os
    import sys

    from common import GOLDEN

    sys.path.insert(0, GOLDEN)
    from make_golden_large import functional, sample_index

    g = dict(np.load(os.path.join(GOLDEN, "cfg3_ops.npz")))
    prob, dec, cs, M = build(g)
    x = operator_input(prob.A.shape[0], False)
    c = cs.r0 @ x
    y = np.zeros_like(x)
    outs = {"Ax": prob.A @ x, "R0x": c, "R0T_c": cs.r0.T @ c, "coarse_solve": cs.lu.solve(c),
            "coarse_correct": O.coarse_correct(cs, x), "local_sum": M.local_sum(x, y, True), "M_shs2": M(x)}
    nu, m0 = int(g["nu"]), int(g["m0"])
    for tag, v in outs.items():
        ref = g[tag]
        idx = sample_index(m0 if tag in ("R0x", "coarse_solve") else nu)
        assert rel(v[idx], ref) <= 1e-12, tag
        assert abs(np.linalg.norm(v) - float(g[tag + "_norm"])) <= 1e-12 * float(g[tag + "_norm"]), tag
        w = functional(len(v))
        assert abs(w @ v - float(g[tag + "_dot"])) <= 1e-12 * np.linalg.norm(w) * float(g[tag + "_norm"]), tag
