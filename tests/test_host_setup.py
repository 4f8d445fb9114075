"""Host-side setup and ABI checks that need no GPU.

* the FDM setup (eigen-pairs, pivoted band LU) emulated in numpy exactly as the
  kernels use it reproduces the oracle's SuperLU solves;
* the box descriptors reproduce the reference's index sets and weights;
* libhelmb200.so loads and exports every symbol include/helmb200.h declares.
"""

import os
import re

import numpy as np
import pytest

import fdm_emulation as E
import helmdd_oracle as O
from paper_2408_03571_b200 import discretization as D
from paper_2408_03571_b200 import fdm_setup as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n,k,problem,p,m", [(65, 20.0, "MP1", 4, 2), (65, 10.0, "MP2", 8, 2),
                                             (129, 30.0, "MP2", 8, 2), (33, 9.0, "MP1", 4, 3),
                                             (17, 2.0, "MP1", 4, 2)])
def test_fdm_emulation_matches_superlu(n, k, problem, p, m):
    prob, dec, cs, M = O.build_shs2(n, k, problem, p, m)
    g = D.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    ours = D.extend(D.partition(g, p), m)
    lc = F.local_classes(g, k, ours.boxes)
    cf = F.coarse_fast(g, k)
    rng = np.random.default_rng(3)
    N = prob.A.shape[0]
    x = rng.standard_normal(N) + (1j * rng.standard_normal(N) if problem == "MP2" else 0)
    c = cs.r0 @ x
    ref = cs.lu.solve(c)
    for refine, strip_refine in ((0, 1), (1, 0), (0, 0)):  # product default first
        got = E.coarse_solve(cf, k, c, refine=refine, strip_refine=strip_refine)
        tol = 1e-12 if (refine, strip_refine) != (0, 0) else 1e-11
        assert np.linalg.norm(got - ref) <= tol * np.linalg.norm(ref), (refine, strip_refine)
    dt = complex if problem == "MP2" else float
    ref = M.local_sum(x.astype(dt), np.zeros(N, dt), True)
    got = E.local_sum(ours, lc, k, x)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_strip_refinement_recovers_accuracy():
    """Sommerfeld coarse solve at m0 = 257: the eigen-space Woodbury step alone leaves a
    strip-supported residual; one strip-refinement pass (exact residual from the band
    pass) brings the solution to the accuracy of a refined solve."""
    g = D.Grid(513, "sommerfeld")
    k = 100.0
    cf = F.coarse_fast(g, k)
    m = cf.m0
    rng = np.random.default_rng(1)
    C = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    ref = E.coarse_solve(cf, k, C.ravel(), refine=2, strip_refine=1)
    err = {sr: np.linalg.norm(E.coarse_solve(cf, k, C.ravel(), refine=0, strip_refine=sr) - ref) / np.linalg.norm(ref)
           for sr in (0, 1)}
    assert err[1] <= 5e-14 and err[1] < 0.2 * err[0], err
    Y = E.fast_solve(cf, C, 0)
    R = C - E.a0_apply(cf, k, Y)
    off = np.delete(R, cf.strip_x, axis=1)
    per_col = lambda X: np.linalg.norm(X) / np.sqrt(X.shape[1])  # noqa: E731
    assert per_col(off) < 0.1 * per_col(R[:, cf.strip_x])  # the residual concentrates on the strips


def test_coarse_pencil_reconstructs_galerkin_matrix():
    """A0 = T0(x)M0 + M0(x)T0 - k^2 M0(x)M0 equals the reference's symmetrised R0 A R0^T."""
    for n, k, problem in [(33, 7.0, "MP2"), (33, 9.0, "MP1")]:
        prob, dec, cs, M = O.build_shs2(n, k, problem, 4, 2)
        g = D.Grid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
        cf = F.coarse_fast(g, k)
        Y = np.random.default_rng(0).standard_normal((cf.m0, cf.m0))
        got = E.a0_apply(cf, k, Y).ravel()
        ref = cs.a0 @ Y.ravel()
        assert np.linalg.norm(got - ref) <= 1e-14 * np.linalg.norm(ref)
        if problem == "MP2":  # y-pencil eigenbasis of the capacitance step: (V^T M0)(M0 V)^T ... = I
            m = cf.m0
            M0 = np.zeros((m, m), dtype=cf.m0b.dtype)
            for d in range(-2, 3):
                i = np.arange(max(0, -d), min(m, m - d))
                M0[i, i + d] = cf.m0b[i, d + 2]
            V = np.linalg.solve(M0, cf.cap_right)
            assert np.abs(cf.cap_left @ V - np.eye(m)).max() < 1e-10


@pytest.mark.parametrize("n,p,m,bc", [(65, 4, 2, "dirichlet"), (65, 8, 2, "sommerfeld"), (33, 4, 3, "sommerfeld"),
                                      (17, 2, 4, "dirichlet"), (17, 4, 0, "sommerfeld")])
def test_boxes_match_reference_decomposition(n, p, m, bc):
    og = O.OGrid(n, bc)
    odec = O.decompose(og, p, m)
    dec = D.extend(D.partition(D.Grid(n, bc), p), m)
    for a, b in zip(odec.index_sets, dec.index_sets):
        assert np.array_equal(a, b)
    for a, b in zip(odec.weights, dec.weights):
        assert np.array_equal(a, b)


def test_band_lu_solves_shifted_pencils():
    g = D.Grid(33, "sommerfeld")
    cf = F.coarse_fast(g, 7.0)
    m = cf.m0
    rng = np.random.default_rng(1)
    G = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    H = E.band_solve(cf.piv, cf.L, cf.U, G)
    for a in (0, m // 2, m - 1):
        S = np.zeros((m, m), complex)
        for d in range(-2, 3):
            i = np.arange(max(0, -d), min(m, m - d))
            S[i, i + d] = cf.t0b[i, d + 2] + cf.shifts[a] * cf.m0b[i, d + 2]
        assert np.linalg.norm(S @ H[:, a] - G[:, a]) <= 1e-12 * np.linalg.norm(G[:, a])


def test_library_exports_every_declared_symbol():
    from paper_2408_03571_b200 import _lib

    lib = _lib.load()
    hdr = open(os.path.join(ROOT, "include", "helmb200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int32_t|int64_t|uint64_t|const char\*)\s+(helm_\w+)\(", hdr, re.M))
    assert declared, "no declarations parsed"
    bound = {s[0] for s in _lib.SYMBOLS}
    assert declared == bound
    for name in declared:
        assert hasattr(lib, name)
    assert lib.helm_abi_version() == _lib.ABI_VERSION


def test_desc_layout_matches_header(tmp_path):
    """ctypes mirror of helm_desc / helm_gmres_report has the C layout (gcc on the header)."""
    import ctypes
    import subprocess

    from paper_2408_03571_b200 import _lib

    structs = {"helm_desc": _lib.HelmDesc, "helm_gmres_report": _lib.HelmGmresReport, "helm_problem": _lib.HelmProblem}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "helmb200.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l}
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py)
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


def test_resonant_subdomain_raises_singular():
    """A k^2 on a subdomain eigenvalue: the reference's splu raises SingularMatrixError
    (linalg.py:76-86); the FDM setup must too instead of dividing by ~0 on the device."""
    import paper_2408_03571_b200 as hb
    from paper_2408_03571_b200.discretization import pencil_1d
    from paper_2408_03571_b200.fdm_setup import _sym_pencil_eig, local_classes

    grid = hb.Grid(17, "dirichlet")
    dec = hb.extend(hb.partition(grid, 2), 2)
    T, w = pencil_1d(grid, 0.0)
    s, L = dec.boxes[0]
    lam, _ = _sym_pencil_eig(T[s:s + L, s:s + L], w[s:s + L])
    k = float(np.sqrt(2 * lam[0]))  # lam_y[0] + lam_x[0] - k^2 = 0 on the first box
    with pytest.raises(hb.SingularMatrixError):
        local_classes(grid, k, dec.boxes)
    local_classes(grid, k * 1.01, dec.boxes)  # off resonance: fine


def test_out_buffer_is_validated():
    """A caller-supplied out buffer is checked before its raw pointer reaches a kernel."""
    import torch

    from paper_2408_03571_b200.operators import _check_out

    ok = torch.empty((2, 10), dtype=torch.complex128)
    _check_out(ok, (2, 10), torch.complex128, ok.device)
    with pytest.raises(TypeError):
        _check_out(torch.empty((2, 10), dtype=torch.float64), (2, 10), torch.complex128, ok.device)
    with pytest.raises(ValueError):
        _check_out(torch.empty((2, 9), dtype=torch.complex128), (2, 10), torch.complex128, ok.device)
    with pytest.raises(ValueError):
        _check_out(torch.empty((10, 2), dtype=torch.complex128).t(), (2, 10), torch.complex128, ok.device)


GENERAL_COARSE = [("MP2", 81, 20.0, "HOCS", 4), ("MP1", 81, 20.0, "HOCS", 4), ("MP2", 81, 20.0, "FOCS", 4),
                  ("MP1", 65, 10.0, "FOCS", 2), ("MP1", 97, 5.0, "HOCS", 16), ("MP2", 129, 30.0, "HOCS", 8),
                  ("MP2", 61, 12.0, "FOCS", 3)]


@pytest.mark.parametrize("problem,n,k,kind,ratio", GENERAL_COARSE)
def test_general_coarse_setup_matches_oracle(problem, n, k, kind, ratio):
    """FOCS / HOCS ratio 4, 8, 16 (coarse.py:84-151): our 1-D P equals the oracle's, and the
    dense fast diagonalisation, refined twice with the banded A0 exactly as coarse_dense.cu does,
    solves the oracle's Galerkin matrix to the SuperLU level."""
    import scipy.sparse as sp

    import paper_2408_03571_b200 as hb
    from paper_2408_03571_b200.fdm_setup import coarse_dense

    bc = "dirichlet" if problem == "MP1" else "sommerfeld"
    grid = hb.Grid(n, bc)
    cs = (hb.build_hocs if kind == "HOCS" else hb.build_focs)(grid, ratio)
    P = cs.restriction_1d()
    og = O.OGrid(n, bc)
    Po = (O.bezier_1d(og, ratio) if kind == "HOCS" else O.hat_1d(og, ratio)).toarray()
    assert np.array_equal(P, Po)
    assert P.shape[0] == cs.coarse_unknowns_per_dim
    cd = coarse_dense(grid, k, P)
    op = O.assemble(og, k, problem)
    R0, a0 = O.galerkin_matrix(og, op.A, ratio, kind)
    m = cd.m0
    c = np.random.default_rng(3).standard_normal(m * m) + (1j * np.random.default_rng(4).standard_normal(m * m)
                                                           if problem == "MP2" else 0)

    # the stencil IS the oracle's (= the reference's) Galerkin matrix, bit for bit
    wd = 2 * cd.bw + 1
    rows, taps = np.nonzero(cd.a0_stencil)
    iy, ix = np.divmod(rows, m)
    dy, dx = np.divmod(taps, wd)
    A0 = sp.csr_matrix((cd.a0_stencil[rows, taps], (rows, (iy + dy - cd.bw) * m + ix + dx - cd.bw)), shape=(m * m, m * m))
    assert (A0 != a0).nnz == 0

    def fdm(C):
        return cd.V @ ((cd.V.T @ C @ cd.V) * cd.invden) @ cd.V.T

    C = c.reshape(m, m)
    Y = fdm(C)
    for _ in range(2):  # coarse_dense.cu: r = C - A0 Y (the stencil), Y += solve(r)
        Y = Y + fdm(C - (a0 @ Y.ravel()).reshape(m, m))
    ref = sp.linalg.splu(sp.csc_matrix(a0)).solve(c)
    assert np.linalg.norm(Y.ravel() - ref) <= 1e-12 * np.linalg.norm(ref)
    # the banded P / P^T tables reproduce P
    Pb = np.zeros_like(P)
    for r in range(m):
        w = cd.p_taps.shape[1]
        cols = cd.p_start[r] + np.arange(w)
        ok = cols < P.shape[1]
        Pb[r, cols[ok]] = cd.p_taps[r, ok]
    assert np.array_equal(Pb, P)


def test_harness_config_mirror(tmp_path):
    """The B200 harness reads the reference's config format and emits its CSV layout
    (harness.py:82-151, 242-263): keys, defaults, errors, warnings."""
    from paper_2408_03571_b200 import harness as Hh

    cfgf = tmp_path / "sweep.cfg"
    cfgf.write_text("problem = mp2\nk = 20, 40\nn = 81, 161\ncoarse = hocs, focs\npreconditioners = shs2\n"
                    "rtol = 1e-6\nprecond_side = left  # comment\n")
    cfg = Hh.parse_config(cfgf)
    assert cfg.problem == "MP2" and cfg.k_list == (20, 40) and cfg.n_list == (81, 161)
    assert cfg.coarse_kinds == ("HOCS", "FOCS") and cfg.gmres.side == "left" and cfg.gmres.rtol == 1e-6
    assert cfg.coarse_ratio == 4 and cfg.overlap == "max" and cfg.cells() == [(20, 81), (40, 161)]
    with pytest.raises(Hh.ConfigError):
        Hh.config_from_dict({"k": "1", "n": "9", "bogus": "1"})
    with pytest.raises(Hh.ConfigError):
        Hh.config_from_dict({"k": "1", "n": "9", "coarse": "XYZ"})
    with pytest.raises(Hh.ConfigError):
        Hh.validate_config(Hh.config_from_dict({"k": "20", "n": "80"}))  # 4 does not divide 79
    (_, _, p, rep, warns), = Hh.validate_config(Hh.config_from_dict({"k": "200", "n": "81"}))
    assert p == 20 and not rep.kappa_h_ok and any("kappa_h" in w for w in warns)
    t1 = Hh.builtin_table(1)
    assert t1.problem == "MP2" and t1.coarse_kinds == ("FOCS", "HOCS") and t1.gmres.side == "left"
    assert Hh.builtin_table(4).coarse_ratio == 16 and Hh.builtin_table(2).problem == "MP1"
    row = Hh.TableRow(k=20, n=81, subdomains=400, fine_nodes=6561, coarse_nodes=441, kappa_h=0.25, kappa_H=1.0,
                      iterations={"HOCS_SHS2": 8, "FOCS_SHS2": "x"})
    out = Hh.emit_csv([row], tmp_path / "t.csv").read_text().splitlines()
    assert out[0] == "k,n,subdomains,fine_nodes,coarse_nodes,kappa_h,kappa_H,HOCS_SHS2,FOCS_SHS2,setup_seconds,solve_seconds"
    assert out[1].startswith("20,81,400,6561,441,0.25,1,8,x,")
    with pytest.raises(ValueError):
        Hh.emit_csv([], tmp_path / "e.csv")
    with pytest.raises(Hh.ConfigError):
        Hh.run_experiment(t1, backend="cpu")


def test_even_n_follows_the_reference():
    """discretization.py:172-173, 183-188: MP-1 needs odd n (same message), MP-2 takes even n with
    the load at the node nearest the centre; coarse.py:78-79: the ratio must divide n - 1."""
    import paper_2408_03571_b200 as hb

    with pytest.raises(ValueError, match="MP1 needs odd n"):
        hb.assemble(hb.Grid(46, "dirichlet"), 8.0, "MP1")
    grid = hb.Grid(64, "sommerfeld")
    prob = hb.assemble(grid, 12.0, "MP2")
    c = (64 - 1) // 2
    assert prob.f[grid.unknown_index(c, c)] == 1.0 / grid.h**2 and np.count_nonzero(prob.f) == 1
    with pytest.raises(ValueError, match="does not divide"):
        hb.build_hocs(grid, 2)
    assert hb.build_focs(grid, 3).ratio == 3
