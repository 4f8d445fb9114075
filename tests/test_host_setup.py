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

    structs = {"helm_desc": _lib.HelmDesc, "helm_gmres_report": _lib.HelmGmresReport}
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
