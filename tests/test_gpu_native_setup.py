"""Native setup (helm_plan_create_problem): the library builds the box classes and
their eigen-pairs (cuSOLVER), the coarse transform eigenvalues, band LU and Woodbury data from the
problem parameters alone.  Checked against the host (numpy/LAPACK) setup and the reference goldens."""

import numpy as np
import pytest
import torch

from common import load_golden, operator_input, rel

pytestmark = pytest.mark.gpu

CASES = [("MP2", 65, 10.0, 8, 2), ("MP1", 65, 20.0, 4, 2), ("MP2", 257, 50.0, 8, 2), ("MP1", 513, 100.0, 16, 2),
         ("MP2", 33, 7.0, 4, "max"), ("MP1", 33, 9.0, 4, 3)]


def make(problem, n, k, p, m, kind="SHS2", setup="native", **kw):
    import paper_2408_03571_b200 as hb

    grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = hb.assemble(grid, k, problem)
    part = hb.partition(grid, p)
    dec = hb.extend_max(part) if m == "max" else hb.extend(part, m)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    return prob, hb.SchwarzPreconditioner(kind, prob.A, dec, cs, setup=setup, **kw)


@pytest.mark.parametrize("problem,n,k,p,m", CASES)
def test_native_setup_matches_host_setup(problem, n, k, p, m):
    for kind in ("SHS2", "AS2", "SAS2"):
        prob, Mn = make(problem, n, k, p, m, kind, "native")
        _, Mh = make(problem, n, k, p, m, kind, "host")
        assert Mn.setup == "native" and Mh.setup == "host"
        x = operator_input(prob.A.N, problem == "MP2")
        c = Mh.restrict(x)
        errs = {"M": rel(Mn(x), Mh(x)), "A0^-1": rel(Mn.coarse_solve(c), Mh.coarse_solve(c)),
                "local": rel(Mn.local_sum(x), Mh.local_sum(x))}
        print(problem, n, k, p, m, kind, {a: f"{b:.1e}" for a, b in errs.items()})
        assert all(v <= 1e-12 for v in errs.values()), errs


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "small_mp2_n65_p8"])
def test_native_setup_matches_reference(name):
    import paper_2408_03571_b200 as hb

    g = load_golden(name)
    prob, M = make(str(g["problem"]), int(g["n"]), float(g["k"]), int(g["p"]), int(g["overlap_layers"]))
    x = operator_input(prob.A.N, str(g["problem"]) == "MP2")
    assert rel(M(x), g["M_shs2"]) <= 1e-12
    assert rel(M.coarse_solve(g["R0x"]), g["coarse_solve"]) <= 1e-12
    b = prob.f
    rep = hb.gmres(prob.A, M, b, hb.GmresConfig(rtol=1e-6, max_iter=1000))
    assert rep.converged and abs(rep.iterations - int(g["gmres_iterations"])) <= 1


def test_native_setup_raw_abi():
    """A C caller: only helm_problem, no host arrays (the ctypes call is what a C program does)."""
    import ctypes

    from paper_2408_03571_b200 import _lib

    lib = _lib.load()
    pr = _lib.HelmProblem(n=129, bc=_lib.HELM_SOMMERFELD, kind=_lib.KINDS["SHS2"], weights_before_solve=0, p=8,
                          overlap_layers=2, coarse_kind=0, ratio=2, k=20.0, strip_refine=-1, refine_steps=-1)
    h = ctypes.c_void_p()
    assert lib.helm_plan_create_problem(ctypes.byref(pr), ctypes.byref(h)) == 0, lib.helm_last_error()
    assert lib.helm_plan_num_unknowns(h) == 129 * 129 and lib.helm_plan_num_coarse(h) == 65 * 65
    ws = ctypes.c_void_p()
    assert lib.helm_workspace_create(h, 1, ctypes.byref(ws)) == 0
    x = torch.ones(129 * 129, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    assert lib.helm_apply_M(h, ws, x.data_ptr(), y.data_ptr(), 1, st) == 0
    torch.cuda.synchronize()
    assert torch.isfinite(y.abs()).all()
    bad = _lib.HelmProblem(n=128, bc=_lib.HELM_SOMMERFELD, kind=2, p=8, overlap_layers=2, ratio=2, k=20.0)
    h2 = ctypes.c_void_p()
    assert lib.helm_plan_create_problem(ctypes.byref(bad), ctypes.byref(h2)) != 0
    assert b"odd" in lib.helm_last_error()
    lib.helm_workspace_destroy(ws)
    lib.helm_plan_destroy(h)
