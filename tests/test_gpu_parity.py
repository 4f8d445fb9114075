"""GPU parity: every operator of the hot path against the reference's own outputs.

The golden fixtures were produced by the unmodified reference (tests/golden/make_golden.py);
inputs are regenerated from the same seeds.  Bars (BASELINE.json north_star):
operator applies <= 1e-12 relative, GMRES iteration counts within +-1, solutions <= 1e-8.
"""

import numpy as np
import pytest
import torch

from common import (accurate_reference_counts, count_matches, golden_names, load_golden, operator_input,
                    random_rhs, raw_reference_counts, reference_count, reference_solution_spread, rel)

pytestmark = pytest.mark.gpu

OP_TOL = 1e-12
X_TOL = 1e-8
# cfg2: the reference's iterate is not reproducible by the reference itself at the 1e-8 level
# (point source on a symmetric domain: rounding breaks the symmetry and GMRES amplifies it;
# tests/test_reference_reproducibility.py measures <= 6e-7 under 1e-15 perturbations of M).
UNREPRODUCIBLE = {"cfg2": 2e-6}
# cfg3 / cfg4a (near-resonant): the reference's own count and iterate move under the choices its
# SPEC leaves open (SuperLU ordering, subdomain order) and with its inner solves made accurate;
# tests/golden/<cfg>_spread.json (make_spread.py) records that spread, and the bars below are
# taken from it (NEAR_RESONANT_BARS): the count within +-1 of the accurate-solve reference counts,
# the iterate within the reference's own solution spread under the SPEC-allowed variations.
NEAR_RESONANT = ("cfg3", "cfg4a")

_cache = {}


def build(name):
    if name in _cache:
        return _cache[name]
    import paper_2408_03571_b200 as hb

    g = load_golden(name)
    n, k, problem, p, m = int(g["n"]), float(g["k"]), str(g["problem"]), int(g["p"]), int(g["overlap_layers"])
    grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = hb.assemble(grid, k, problem)
    dec = hb.extend(hb.partition(grid, p), m)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    Ms = {kind: hb.SchwarzPreconditioner(kind, prob.A, dec, cs, max_batch=4) for kind in ("SHS2", "AS2", "SAS2")}
    _cache[name] = (g, prob, Ms)
    return _cache[name]


VEC_CASES = golden_names(store_vectors=True)
RUN_CASES = golden_names(store_vectors=False)


@pytest.mark.parametrize("name", VEC_CASES)
def test_operators_match_reference(name):
    g, prob, Ms = build(name)
    M = Ms["SHS2"]
    x = operator_input(prob.A.N, prob.problem == "MP2")
    errs = {}
    if "Ax" in g:
        errs["A x"] = rel(prob.A @ x, g["Ax"])
    errs["R0 x"] = rel(M.restrict(x), g["R0x"])
    errs["A0^-1 c"] = rel(M.coarse_solve(g["R0x"]), g["coarse_solve"])
    if "R0T_c" in g:
        errs["R0^T c"] = rel(M.prolong(g["R0x"]), g["R0T_c"])
        errs["coarse_correct"] = rel(M.coarse_correct(x), g["coarse_correct"])
        errs["local_sum"] = rel(M.local_sum(x, weighted=True), g["local_sum"])
    errs["M SHS2"] = rel(M(x), g["M_shs2"])
    if "M_as2" in g:
        errs["M AS2"] = rel(Ms["AS2"](x), g["M_as2"])
        errs["M SAS2"] = rel(Ms["SAS2"](x), g["M_sas2"])
    bad = {k: v for k, v in errs.items() if not v <= OP_TOL}
    print(name, {k: f"{v:.1e}" for k, v in errs.items()})
    assert not bad, bad


@pytest.mark.parametrize("name", VEC_CASES)
def test_gmres_matches_reference(name):
    import paper_2408_03571_b200 as hb

    g, prob, Ms = build(name)
    b = prob.f if str(g["gmres_rhs"]) == "point" else random_rhs(prob.A.N)
    rep = hb.gmres(prob.A, Ms["SHS2"], b, hb.GmresConfig(rtol=1e-6, max_iter=1000))
    assert rep.converged == bool(g["gmres_converged"])
    raw = reference_count(name, g)
    assert count_matches(rep.iterations, raw), (rep.iterations, raw)
    xe = rel(rep.x, g["gmres_x"])
    print(name, rep.iterations, raw, f"x {xe:.1e}")
    assert rep.final_residual <= 1e-6
    if name in UNREPRODUCIBLE:
        # the reference itself moves by >1e-8 here under 1e-15 perturbations of M
        # (tests/test_reference_reproducibility.py): bound by its own spread instead
        assert xe <= UNREPRODUCIBLE[name]
    else:
        assert xe <= X_TOL
        h, hr = rep.residual_history, g["gmres_history"]
        assert np.all(np.abs(h - hr) <= 1e-6 * np.maximum(hr, 1e-30) + 1e-12)


@pytest.mark.parametrize("name", RUN_CASES)
def test_gmres_large_configs(name):
    """BASELINE configs 3 and 4: iteration counts, residual histories, sampled solutions.
    Config 4(b) (random RHS) does not converge within 1000 iterations; its golden is the
    reference's first 100 iterations, compared estimate by estimate and on the iterate."""
    import paper_2408_03571_b200 as hb

    g, prob, Ms = build(name)
    b = prob.f if str(g["gmres_rhs"]) == "point" else random_rhs(prob.A.N)
    cap = int(g["gmres_cap"]) if "gmres_cap" in g else 1000
    rep = hb.gmres(prob.A, Ms["SHS2"], b, hb.GmresConfig(rtol=1e-6, max_iter=cap))
    raw = reference_count(name, g)
    stride = int(g["gmres_x_sample_stride"])
    xe = rel(rep.x[::stride], g["gmres_x_sample"])
    print(name, rep.iterations, raw, f"x(sample) {xe:.1e}", f"{rep.wall_seconds:.2f}s")
    if not bool(g["gmres_converged"]):  # fixed-length run: the same iterates
        assert not rep.converged and rep.iterations == raw
        h, hr = rep.residual_history, g["gmres_history"]
        assert np.all(np.abs(h - hr) <= 1e-9 * hr), np.max(np.abs(h - hr) / hr)
        assert abs(rep.final_residual - float(g["gmres_final_residual"])) <= 1e-9 * float(g["gmres_final_residual"])
        assert xe <= X_TOL
        return
    assert rep.converged and rep.final_residual <= 1e-6
    if name not in NEAR_RESONANT:
        assert count_matches(rep.iterations, raw) and xe <= X_TOL, (rep.iterations, raw, xe)
        return
    acc = accurate_reference_counts(name)
    spread = reference_solution_spread(name, g)
    print(name, "reference raw counts", raw_reference_counts(name, g), "accurate-solve counts", acc,
          f"reference solution spread {spread:.1e}")
    assert acc and acc[0] - 1 <= rep.iterations <= acc[-1] + 1, (rep.iterations, acc)
    assert spread > 0 and xe <= spread, (xe, spread)


@pytest.mark.parametrize("name", NEAR_RESONANT)
@pytest.mark.xfail(strict=True, reason="known gap: the reference's raw count (cfg3 100, cfg4a 373) is set by "
                   "the ~1e-13 rounding of its SuperLU solves; with accurate inner solves the reference itself "
                   "gives 95-97 / 363-366 (tests/golden/<cfg>_spread.json, DESIGN.md §5)")
def test_raw_reference_count_near_resonant(name):
    import paper_2408_03571_b200 as hb

    g, prob, Ms = build(name)
    rep = hb.gmres(prob.A, Ms["SHS2"], prob.f, hb.GmresConfig(rtol=1e-6, max_iter=1000))
    assert count_matches(rep.iterations, reference_count(name, g)), (rep.iterations, reference_count(name, g))


def test_batched_apply_matches_single():
    g, prob, Ms = build(VEC_CASES[0])
    M = Ms["SHS2"]
    rng = np.random.default_rng(7)
    X = rng.standard_normal((3, prob.A.N))
    if prob.problem == "MP2":
        X = X + 1j * rng.standard_normal((3, prob.A.N))
    Y = M(torch.from_numpy(X).cuda()).cpu().numpy()
    for i in range(3):  # batched kernels pair/sum rows differently: rounding-level differences only
        assert rel(Y[i], M(X[i])) <= 1e-14


def test_zero_maps_to_zero():
    g, prob, Ms = build(VEC_CASES[0])
    for M in Ms.values():
        assert np.all(M(np.zeros(prob.A.N)) == 0.0)


def test_dimension_mismatch_rejected():
    g, prob, Ms = build(VEC_CASES[0])
    with pytest.raises(ValueError):
        Ms["SHS2"](np.ones(prob.A.N + 1))


def test_zero_rhs_rejected():
    import paper_2408_03571_b200 as hb

    g, prob, Ms = build(VEC_CASES[0])
    with pytest.raises(ValueError):
        hb.gmres(prob.A, Ms["SHS2"], np.zeros(prob.A.N, dtype=prob.A.dtype))


def test_reference_csr_accepted_through_structure_guard():
    import paper_2408_03571_b200 as hb
    import helmdd_oracle as O

    g, prob, Ms = build("cfg1")
    op = O.assemble(O.OGrid(65, "dirichlet"), 20.0, "MP1")
    dec = hb.extend(hb.partition(prob.grid, 4), 2)
    M = hb.SchwarzPreconditioner("SHS2", op.A, dec, hb.build_hocs(prob.grid, 2))
    x = operator_input(prob.A.N, False)
    assert rel(M(x), g["M_shs2"]) <= OP_TOL
    bad = op.A.copy()
    bad[5, 5] += 1.0
    with pytest.raises(ValueError):
        hb.SchwarzPreconditioner("SHS2", bad, dec, hb.build_hocs(prob.grid, 2))


def test_pipelined_host_apply_matches_device():
    """Pinned host batch -> pinned host result (PCIe copies overlapped with the kernels, chunked)
    equals the device-resident batched apply bit for bit."""
    import paper_2408_03571_b200 as hb

    grid = hb.Grid(65, "sommerfeld")
    prob = hb.assemble(grid, 10.0, "MP2")
    dec = hb.extend(hb.partition(grid, 8), 2)
    M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, hb.build_hocs(grid, 2), max_batch=19)
    rng = np.random.default_rng(11)
    X = torch.from_numpy(rng.standard_normal((19, prob.A.N)) + 1j * rng.standard_normal((19, prob.A.N)))
    Xh = X.pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    M.apply(Xh, out=Yh)
    ref = torch.empty(19, prob.A.N, dtype=torch.complex128, device="cuda")
    for lo in range(0, 19, M.PIPE_CHUNK):  # same chunking -> same batched kernels
        hi = min(19, lo + M.PIPE_CHUNK)
        ref[lo:hi] = M(X[lo:hi].cuda())
    assert torch.equal(Yh, ref.cpu())


@pytest.mark.parametrize("n,k,p", [(257, 50.0, 8), (513, 100.0, 16)])
def test_segmented_band_solve_matches_lane_recurrence(n, k, p):
    """Small batches run the coarse band solves as a segmented linear recurrence
    (band_seg.cu), larger ones one lane per mode (band.cu): same solve, different
    association.  Both must agree to rounding, and the coarse solve must satisfy A0 y = c."""
    import paper_2408_03571_b200 as hb

    grid = hb.Grid(n, "sommerfeld")
    prob = hb.assemble(grid, k, "MP2")
    dec = hb.extend(hb.partition(grid, p), 2)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, max_batch=8)
    import scipy.sparse as sp
    import helmdd_oracle as O  # checker only: A0 = R0 A R0^T

    og = O.OGrid(n, "sommerfeld")
    oprob = O.assemble(og, k, "MP2")
    P1 = O.bezier_1d(og, 2)
    r0 = sp.kron(P1, P1, format="csr").astype(complex)
    a0 = (r0 @ oprob.A @ r0.T).tocsr()
    rng = np.random.default_rng(3)
    C = rng.standard_normal((8, M.N0)) + 1j * rng.standard_normal((8, M.N0))
    Yb = M.coarse_solve(torch.from_numpy(C).cuda()).cpu().numpy()  # batch 8: lane recurrence
    for i in (0, 5):
        y1 = M.coarse_solve(C[i])  # batch 1: segmented recurrence
        assert rel(y1, Yb[i]) <= 1e-13
        assert np.linalg.norm(a0 @ y1 - C[i]) / np.linalg.norm(C[i]) <= 1e-12


def test_cgs2_every_basis_size_launches():
    """The CGS2 kernels size their shared memory by the basis length: every length up to a
    long run (including the 48 KB opt-in boundary at 384 vectors) must launch, and the new
    vector must come out orthonormal to the basis."""
    import paper_2408_03571_b200 as hb

    grid = hb.Grid(65, "sommerfeld")
    prob = hb.assemble(grid, 10.0, "MP2")
    M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 8), 2), hb.build_hocs(grid, 2))
    lib, pl = M.plan.lib, M.plan
    N = M.N
    g = torch.Generator(device="cuda").manual_seed(0)
    for j in (0, 7, 31, 216, 217, 383, 384, 600):
        Q, _ = torch.linalg.qr(torch.randn(N, j + 1, dtype=torch.complex128, device="cuda", generator=g))
        V = torch.cat([Q.T.contiguous(), torch.randn(1, N, dtype=torch.complex128, device="cuda", generator=g)])
        h = torch.empty(j + 2, dtype=torch.complex128, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        assert lib.helm_cgs2(pl.handle, pl.ws, V.data_ptr(), j, h.data_ptr(), st) == 0, lib.helm_last_error()
        torch.cuda.synchronize()
        w = V[j + 1]
        assert abs(torch.linalg.vector_norm(w).item() - 1.0) < 1e-12
        assert torch.abs(V[: j + 1].conj() @ w).max().item() < 1e-12


@pytest.mark.parametrize("problem,n,k,p", [("MP2", 65, 10.0, 8), ("MP1", 65, 12.0, 4)])
@pytest.mark.parametrize("kind", ["AS2", "SAS2", "SHS2"])
def test_weights_before_solve_matches_oracle(problem, n, k, p, kind):
    """schwarz.py:69-70 (weights applied before the local solves) for every kind."""
    import helmdd_oracle as O  # checker only
    import paper_2408_03571_b200 as hb

    grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = hb.assemble(grid, k, problem)
    dec = hb.extend(hb.partition(grid, p), 2)
    M = hb.SchwarzPreconditioner(kind, prob.A, dec, hb.build_hocs(grid, 2), weights_before_solve=True)
    oprob, odec, ocs, _ = O.build_shs2(n, k, problem, p, 2)
    oM = O.OSchwarz(kind, oprob.A, odec, ocs, weights_before_solve=True)
    x = operator_input(prob.A.N, problem == "MP2")
    assert rel(M(x), oM(x)) <= OP_TOL


@pytest.mark.parametrize("problem,n,k,p", [("MP2", 65, 10.0, 8), ("MP1", 65, 20.0, 4)])
def test_left_preconditioned_gmres_matches_oracle(problem, n, k, p):
    """Left preconditioning (gmres.py:79-85,154: stops on the preconditioned estimate):
    same count, history and solution as the oracle."""
    import helmdd_oracle as O  # checker only
    import paper_2408_03571_b200 as hb

    grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = hb.assemble(grid, k, problem)
    M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, p), 2), hb.build_hocs(grid, 2))
    oprob, _, _, oM = O.build_shs2(n, k, problem, p, 2)
    rep = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-7, max_iter=200, side="left"))
    orep = O.gmres(oprob.A, oM, oprob.f, 1e-7, 200, side="left")
    assert rep.converged == orep.converged and rep.iterations == orep.iterations
    assert np.all(np.abs(rep.residual_history - orep.residual_history) <= 1e-6 * orep.residual_history + 1e-14)
    assert rel(rep.x, orep.x) <= X_TOL


def test_compact_band_factors_match_the_general_path(monkeypatch):
    """No pivot taken: the plan stores U rows of 3 entries and skips the pivot reads
    (PlanDev::band_nopiv).  The skipped terms are exact zeros, so M^-1 is bitwise the same as
    with the general 5-entry rows and pivots (HELM_BAND_NOPIV=0), at batch 1 (segmented band
    solve) and batch 6 (lane-per-mode band solve)."""
    import paper_2408_03571_b200 as hb

    grid = hb.Grid(257, "sommerfeld")
    prob = hb.assemble(grid, 50.0, "MP2")
    dec = hb.extend(hb.partition(grid, 8), 2)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    rng = np.random.default_rng(3)
    X = torch.from_numpy(rng.standard_normal((6, prob.A.N)) + 1j * rng.standard_normal((6, prob.A.N))).cuda()
    M1 = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, max_batch=6)
    monkeypatch.setenv("HELM_BAND_NOPIV", "0")
    M0 = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, max_batch=6)
    monkeypatch.delenv("HELM_BAND_NOPIV")
    for Xb in (X[:1], X):
        assert torch.equal(M1(Xb), M0(Xb))


@pytest.mark.parametrize("problem,n,k,p", [("MP2", 33, 10.0, 4), ("MP1", 33, 6.0, 4), ("MP2", 65, 15.0, 4)])
def test_maximal_overlap_matches_oracle(problem, n, k, p):
    """extend_max (decomposition.py:106-108,137-139: m = c // 2, the largest overlap with at most
    two boxes per node per axis) on the device against the CPU oracle: every
    preconditioner kind to 1e-12, SHS2-GMRES count and solution."""
    import sys, os

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import helmdd_oracle as O  # checker only
    import paper_2408_03571_b200 as hb

    grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = hb.assemble(grid, k, problem)
    part = hb.partition(grid, p)
    dec = hb.extend_max(part)
    m = hb.max_overlap_layers(part)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    x = operator_input(prob.A.N, problem == "MP2")
    for kind in ("SHS2", "AS2", "SAS2"):
        M = hb.SchwarzPreconditioner(kind, prob.A, dec, cs)
        oprob, odec, ocs, oM = O.build_shs2(n, k, problem, p, m, kind=kind)
        assert rel(M(x), oM(x)) <= OP_TOL, (kind, rel(M(x), oM(x)))
    M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs)
    oprob, odec, ocs, oM = O.build_shs2(n, k, problem, p, m)
    rep = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-6, max_iter=500))
    orep = O.gmres(oprob.A, oM, oprob.f, 1e-6, 500)
    assert rep.converged and rep.iterations == orep.iterations, (rep.iterations, orep.iterations)
    assert rel(rep.x, orep.x) <= X_TOL


@pytest.mark.parametrize("name", ["cfg1", "small_mp2_n65_p8", "cfg2"])
def test_reference_gmres_drives_device_preconditioner(name):
    """The drop-in as INTEGRATION.md §1 wires it: the reference's own GMRES loop (the oracle's
    restatement of gmres.py:65-177, numpy vectors, the assembled CSR A) calling the device
    SchwarzPreconditioner for every M^{-1} apply (host->device->host per call).  Same count as the
    reference's golden run (+-1) and the device GMRES, same solution."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import helmdd_oracle as O  # the reference's loop, restated (checker)

    import paper_2408_03571_b200 as hb

    g, prob, Ms = build(name)
    n, k, problem = int(g["n"]), float(g["k"]), str(g["problem"])
    oprob = O.assemble(O.OGrid(n, "dirichlet" if problem == "MP1" else "sommerfeld"), k, problem)
    b = oprob.f if str(g["gmres_rhs"]) == "point" else random_rhs(oprob.A.shape[0])
    rep = O.gmres(oprob.A, Ms["SHS2"], b, 1e-6, 1000)  # M: the device preconditioner, numpy in / out
    dev = hb.gmres(prob.A, Ms["SHS2"], b, hb.GmresConfig(rtol=1e-6, max_iter=1000))
    raw = reference_count(name, g)
    print(name, "reference loop + device M:", rep.iterations, "device GMRES:", dev.iterations, "reference:", raw)
    assert rep.converged and count_matches(rep.iterations, raw)
    assert abs(rep.iterations - dev.iterations) <= 1
    tol = UNREPRODUCIBLE.get(name, X_TOL)
    assert rel(rep.x, g["gmres_x"]) <= tol


@pytest.mark.parametrize("problem,n,k,p,wbs", [("MP2", 65, 10.0, 4, False), ("MP2", 257, 50.0, 8, False),
                                                ("MP2", 257, 50.0, 8, True), ("MP1", 65, 20.0, 4, False),
                                                ("MP1", 129, 30.0, 4, True)])
def test_fast_sine_and_edge_boxes_match_dense_path(monkeypatch, problem, n, k, p, wbs):
    """The middle-pencil boxes (fast sine transforms, local_dst.cu) and the MP-2 edge boxes (sine
    transform + one tridiagonal solve per sine mode) against the DMMA / dense box kernels
    (HELM_DST=0, HELM_EDGE=0) and the CPU oracle: the one-level sum and every preconditioner kind
    to 1e-12, at batch 1, 3 (an odd tail of the 2-slot CTAs) and 6."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import helmdd_oracle as O
    import paper_2408_03571_b200 as hb

    grid = hb.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = hb.assemble(grid, k, problem)
    dec = hb.extend(hb.partition(grid, p), 2)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    oprob, odec, ocs, _ = O.build_shs2(n, k, problem, p, 2)
    rng = np.random.default_rng(5)
    shape = (6, prob.A.N)
    Xn = rng.standard_normal(shape) + (1j * rng.standard_normal(shape) if problem == "MP2" else 0.0)
    X = torch.from_numpy(Xn).cuda()
    for kind in ("SHS2", "AS2", "SAS2"):
        Mf = hb.SchwarzPreconditioner(kind, prob.A, dec, cs, max_batch=6, weights_before_solve=wbs)
        monkeypatch.setenv("HELM_DST", "0")
        monkeypatch.setenv("HELM_EDGE", "0")
        Md = hb.SchwarzPreconditioner(kind, prob.A, dec, cs, max_batch=6, weights_before_solve=wbs)
        monkeypatch.delenv("HELM_DST")
        monkeypatch.delenv("HELM_EDGE")
        for Xb in (X[:1], X[:3], X):
            yf, yd = Mf(Xb), Md(Xb)
            assert (torch.linalg.norm(yf - yd) / torch.linalg.norm(yd)).item() <= 1e-12, (kind, Xb.shape[0])
        oM = O.OSchwarz(kind, oprob.A, odec, ocs, weights_before_solve=wbs)
        ref = oM(Xn[1])
        assert rel(Mf(X[1:2])[0].cpu().numpy(), ref) <= 1e-12, kind
