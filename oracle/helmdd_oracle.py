"""CPU oracle for the GMRES + two-level Bezier-Schwarz hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package ``helmdd``
(arXiv 2408.03571, ``/root/reference/pkg/src/helmdd``).  It exists so that the
GPU path can be checked on machines where the reference is not installed (the
GPU box).  Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline``
/ ``--impl reference`` legs of ``bench.py`` may import it, and only as the
checker or the timed CPU baseline — never as a fallback of the product path.

Parity pin: ``tests/golden/make_golden.py`` imports the real reference in the
build container and records its outputs as fixtures under ``tests/golden``;
``tests/test_oracle_golden.py`` checks this module against them (operators to
1e-12 relative, GMRES iteration counts exactly).  The reference's arithmetic is
third-party (scipy SuperLU / CSR matvec, numpy BLAS; versions unpinned in
``pkg/pyproject.toml:10-13``); this restatement calls the same scipy routines,
so it is the same algorithm on the same library.

Every function cites the reference lines it restates.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

# --------------------------------------------------------------------------
# grid + assembly  (discretization.py:36-93, 130-191)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class OGrid:
    """Node grid; unknowns are interior nodes (Dirichlet) or all nodes (Sommerfeld).

    discretization.py:36-84 — h = 1/(n-1), unknown index row-major in y, x fastest.
    """

    n: int
    bc: str

    @property
    def h(self) -> float:
        return 1.0 / (self.n - 1)

    @property
    def lo(self) -> int:  # discretization.py:62-64
        return 1 if self.bc == "dirichlet" else 0

    @property
    def nu(self) -> int:  # unknowns per dimension, discretization.py:66-68
        return self.n - 2 if self.bc == "dirichlet" else self.n

    @property
    def N(self) -> int:
        return self.nu * self.nu

    def index(self, ix, iy):  # discretization.py:74-77
        return (np.asarray(iy) - self.lo) * self.nu + (np.asarray(ix) - self.lo)


def _lap1d(m: int) -> sp.csr_matrix:
    """(-1, 2, -1) tridiagonal — discretization.py:130-133."""
    e = np.ones(m)
    return sp.diags([-e[:-1], 2.0 * e, -e[:-1]], [-1, 0, 1], format="csr")


def sommerfeld_1d(n: int, k: float, h: float) -> sp.csr_matrix:
    """Ghost-point Sommerfeld 1-D operator with halved end rows — discretization.py:136-148.

    End rows: (1, -1)/h^2 - i k/h on the diagonal; interior rows (-1, 2, -1)/h^2.
    """
    d = np.full(n, 2.0 / h**2, dtype=complex)
    d[0] = d[-1] = 1.0 / h**2 - 1j * k / h
    off = np.full(n - 1, -1.0 / h**2, dtype=complex)
    return sp.diags([off, d, off], [-1, 0, 1], format="csr")


def end_weights_1d(n: int) -> np.ndarray:
    """W = diag(1/2, 1, ..., 1, 1/2) — discretization.py:151-154."""
    w = np.ones(n)
    w[[0, -1]] = 0.5
    return w


def pencil_1d(grid: OGrid, k: float):
    """The 1-D pieces (T, w) with A = T(x)W + W(x)T - k^2 W(x)W (W = I for MP-1)."""
    if grid.bc == "dirichlet":
        return (_lap1d(grid.nu) / grid.h**2).tocsr(), np.ones(grid.nu)
    return sommerfeld_1d(grid.n, k, grid.h), end_weights_1d(grid.n)


@dataclass
class OProblem:
    grid: OGrid
    k: float
    problem: str
    A: sp.csr_matrix
    f: np.ndarray


def assemble(grid: OGrid, k: float, problem: str) -> OProblem:
    """MP-1 / MP-2 matrices and centre point load — discretization.py:157-191."""
    if problem not in ("MP1", "MP2"):
        raise ValueError(f"unknown problem {problem!r}")
    if (problem == "MP1") != (grid.bc == "dirichlet"):
        raise ValueError("problem/boundary mismatch")
    T, w = pencil_1d(grid, k)
    if problem == "MP1":
        if grid.n % 2 == 0:
            raise ValueError("MP1 needs odd n")
        I = sp.identity(grid.nu, format="csr")
        A = sp.kron(T, I) + sp.kron(I, T) - k**2 * sp.identity(grid.N)  # :171-177
        f = np.zeros(grid.N)
    else:
        W = sp.diags(w)
        A = sp.kron(T, W) + sp.kron(W, T) - k**2 * sp.kron(W, W)  # :181-184
        f = np.zeros(grid.N, dtype=complex)
    c = (grid.n - 1) // 2
    f[grid.index(c, c)] = 1.0 / grid.h**2  # :178-180, :186-188
    A = sp.csr_matrix(A)
    A.sort_indices()
    return OProblem(grid, k, problem, A, f)


# --------------------------------------------------------------------------
# decomposition  (decomposition.py:66-160)
# --------------------------------------------------------------------------


def box_interval(grid: OGrid, a: int, c: int, m: int):
    """Node interval of 1-D box a with m overlap layers — decomposition.py:66-79."""
    if m == 0:
        lo, hi = a * c + (1 if a > 0 else 0), (a + 1) * c
    else:
        lo, hi = a * c - (m - 1), (a + 1) * c + (m - 1)
    return max(lo, grid.lo), min(hi, grid.lo + grid.nu - 1)


@dataclass
class ODecomposition:
    grid: OGrid
    p: int
    m: int
    index_sets: list
    weights: list
    multiplicity: np.ndarray

    @property
    def c(self) -> int:
        return (self.grid.n - 1) // self.p


def decompose(grid: OGrid, p: int, m: int) -> ODecomposition:
    """partition(grid, p) then extend(part, m) — decomposition.py:89-103, 111-134.

    Boxes are enumerated ay-major (decomposition.py:118-122); weights are the
    inverse multiplicities (decomposition.py:123-133).
    """
    if (grid.n - 1) % p:
        raise ValueError("p does not divide the cell count")
    c = (grid.n - 1) // p
    ivs = [box_interval(grid, a, c, m) for a in range(p)]
    sets = []
    for ylo, yhi in ivs:
        for xlo, xhi in ivs:
            iy, ix = np.mgrid[ylo : yhi + 1, xlo : xhi + 1]
            sets.append(grid.index(ix, iy).ravel())
    mult = np.bincount(np.concatenate(sets), minlength=grid.N).astype(float)
    return ODecomposition(grid, p, m, sets, [1.0 / mult[s] for s in sets], mult)


# --------------------------------------------------------------------------
# coarse space  (coarse.py:102-174)
# --------------------------------------------------------------------------


def bezier_1d(grid: OGrid, ratio: int) -> sp.csr_matrix:
    """Composed one-level (1,4,6,4,1)/8 stride-2 restrictions — coarse.py:102-133.

    Out-of-range taps are dropped (coarse.py:14-15); Dirichlet levels keep
    only interior nodes on both sides (coarse.py:111-120).
    """
    taps = np.array([1.0, 4.0, 6.0, 4.0, 1.0]) / 8.0
    op, nf = None, grid.n
    for _ in range(int(round(np.log2(ratio)))):
        M = (nf + 1) // 2
        I = np.arange(M)[:, None]
        i = 2 * I + np.arange(-2, 3)[None, :]
        wv = np.broadcast_to(taps, i.shape)
        if grid.bc == "dirichlet":
            keep = (I >= 1) & (I <= M - 2) & (i >= 1) & (i <= nf - 2)
            S = sp.csr_matrix(
                (wv[keep], ((I + 0 * i)[keep] - 1, i[keep] - 1)), shape=(M - 2, nf - 2)
            )
        else:
            keep = (i >= 0) & (i < nf)
            S = sp.csr_matrix((wv[keep], ((I + 0 * i)[keep], i[keep])), shape=(M, nf))
        op = S if op is None else S @ op
        nf = M
    op = sp.csr_matrix(op)
    op.sum_duplicates()
    return op


def hat_1d(grid: OGrid, ratio: int) -> sp.csr_matrix:
    """Bilinear hat restriction (FOCS) — coarse.py:84-99."""
    r, n = ratio, grid.n
    M = (n - 1) // r + 1
    J = np.arange(M)[:, None]
    d = np.arange(-r + 1, r)[None, :]
    i = r * J + d
    keep = (i >= 0) & (i < n)
    vals = np.broadcast_to(1.0 - np.abs(d) / r, i.shape)
    P = sp.csr_matrix((vals[keep], ((J + 0 * d)[keep], i[keep])), shape=(M, n))
    if grid.bc == "dirichlet":
        P = P[1:-1, 1:-1]
    return sp.csr_matrix(P)


@dataclass
class OCoarse:
    r0: sp.csr_matrix
    a0: sp.csr_matrix
    lu: object


def galerkin_matrix(grid: OGrid, A: sp.csr_matrix, ratio: int = 2, kind: str = "HOCS"):
    """(R0, A0): build_hocs/build_focs + the symmetrised triple product of galerkin —
    coarse.py:136-139, 154-165 (no factorisation)."""
    P = bezier_1d(grid, ratio) if kind == "HOCS" else hat_1d(grid, ratio)
    R0 = sp.kron(P, P, format="csr")
    R0.sort_indices()
    r0c = R0.astype(A.dtype)
    B = sp.csr_matrix(r0c @ A @ r0c.T)
    a0 = ((B + B.T) * 0.5).tocsr()
    a0.sort_indices()
    return R0, a0


def coarse_space(grid: OGrid, A: sp.csr_matrix, ratio: int = 2, kind: str = "HOCS") -> OCoarse:
    """build_hocs/build_focs + galerkin — coarse.py:136-167 (symmetrised R0 A R0^T, SuperLU)."""
    R0, a0 = galerkin_matrix(grid, A, ratio, kind)
    return OCoarse(R0, a0, splu(sp.csc_matrix(a0)))


def coarse_correct(cs: OCoarse, r: np.ndarray, refine: int = 0) -> np.ndarray:
    """R0^T A0^{-1} R0 r — coarse.py:170-174.

    refine > 0 adds iterative-refinement steps with the same SuperLU factor (NOT in the
    reference; used to measure how the reference's GMRES counts depend on the rounding of
    its coarse solve, tests/golden/make_refined.py)."""
    c = cs.r0 @ r
    y = cs.lu.solve(c)
    for _ in range(refine):
        y = y + cs.lu.solve(c - cs.a0 @ y)
    return cs.r0.T @ y


# --------------------------------------------------------------------------
# Schwarz preconditioners  (schwarz.py:34-103)
# --------------------------------------------------------------------------


class OSchwarz:
    """AS2 / SAS2 / SHS2 applications with exact SuperLU local solves — schwarz.py:31-103."""

    def __init__(self, kind: str, A, dec: ODecomposition, cs: OCoarse, weights_before_solve=False,
                 coarse_refine: int = 0):
        if kind not in ("AS2", "SAS2", "SHS2"):
            raise ValueError(kind)
        self.kind, self.A, self.dec, self.cs = kind, A, dec, cs
        self.wbs = weights_before_solve
        self.coarse_refine = coarse_refine
        # local principal submatrices R_i A R_i^T, factorised once (schwarz.py:55-59)
        self.lus = [splu(sp.csc_matrix(A[s][:, s])) for s in dec.index_sets]

    def local_sum(self, x: np.ndarray, out: np.ndarray, weighted: bool) -> np.ndarray:
        """sum_i R_i^T [D_i] A_i^{-1} [D_i] R_i x accumulated into out — schwarz.py:64-74."""
        for s, w, lu in zip(self.dec.index_sets, self.dec.weights, self.lus):
            xi = x[s]
            if weighted and self.wbs:
                out[s] += lu.solve(w * xi)
            elif weighted:
                out[s] += w * lu.solve(xi)
            else:
                out[s] += lu.solve(xi)
        return out

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x, dtype=np.result_type(np.asarray(x).dtype, self.A.dtype))  # :94
        if x.shape[0] != self.A.shape[0]:
            raise ValueError("dimension mismatch")  # :95-96
        z = coarse_correct(self.cs, x, self.coarse_refine)
        if self.kind == "AS2":  # :76-79
            return self.local_sum(x, z, weighted=False)
        if self.kind == "SAS2":  # :81-84
            return self.local_sum(x, z, weighted=True)
        d = x - self.A @ z  # SHS2 :86-91
        return self.local_sum(d, z.copy(), weighted=True)

    __call__ = apply


def build_shs2(n: int, k: float, problem: str, p: int, m: int = 2, ratio: int = 2, kind="SHS2", coarse="HOCS"):
    """The S1 call stack of SURVEY §3 (README.md:112-121 with extend(part, m), build_hocs /
    build_focs(grid, ratio)); m = "max" is extend_max (decomposition.py:137-139)."""
    grid = OGrid(n, "dirichlet" if problem == "MP1" else "sommerfeld")
    prob = assemble(grid, k, problem)
    if m == "max":
        m = ((n - 1) // p) // 2
    dec = decompose(grid, p, m)
    cs = coarse_space(grid, prob.A, ratio, coarse)
    return prob, dec, cs, OSchwarz(kind, prob.A, dec, cs)


# --------------------------------------------------------------------------
# GMRES  (gmres.py:29-177)
# --------------------------------------------------------------------------


@dataclass
class OReport:
    iterations: int
    converged: bool
    residual_history: np.ndarray
    final_residual: float
    breakdown: bool = False
    wall_seconds: float = 0.0
    x: np.ndarray | None = field(default=None, repr=False)


def _op(f):
    if f is None:
        return lambda v: v
    return f if callable(f) else (lambda v: f @ v)


def gmres(A, M, b, rtol=1e-7, max_iter=100, side="right") -> OReport:
    """Unrestarted GMRES, MGS + one conditional re-orthogonalisation, Givens QR — gmres.py:65-177."""
    t0 = time.perf_counter()
    Aop, Mop = _op(A), _op(M)
    b = np.asarray(b)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        raise ValueError("right-hand side must be nonzero")  # :76-77
    left = side == "left"
    r0 = Mop(b) if left else b
    beta = np.linalg.norm(r0)
    v0 = r0 / beta
    w = Mop(Aop(v0)) if left else Aop(Mop(v0))  # :85
    dt = np.result_type(v0.dtype, w.dtype)
    V = np.zeros((max_iter + 1, b.shape[0]), dt)
    H = np.zeros((max_iter + 1, max_iter), dt)
    cs_, sn_ = np.zeros(max_iter, dt), np.zeros(max_iter, dt)
    g = np.zeros(max_iter + 1, dt)
    V[0], g[0] = v0, beta
    hist = [1.0]

    def solution(j):  # :98-105
        R, rhs = H[: j + 1, : j + 1], g[: j + 1]
        try:
            y = np.linalg.solve(R, rhs)
        except np.linalg.LinAlgError:
            y = np.linalg.lstsq(R, rhs, rcond=None)[0]
        u = V[: j + 1].T @ y
        return u if left else Mop(u)

    for j in range(max_iter):
        if j:
            w = (Mop(Aop(V[j])) if left else Aop(Mop(V[j]))).astype(dt, copy=False)
        for i in range(j + 1):  # MGS :113-116
            hij = np.vdot(V[i], w)
            H[i, j] = hij
            w = w - hij * V[i]
        proj = V[: j + 1].conj() @ w  # :118-122
        wn = np.linalg.norm(w)
        if np.abs(proj).max() > 1e-8 * max(wn, np.finfo(float).tiny):
            H[: j + 1, j] += proj
            w = w - proj @ V[: j + 1]
        hn = np.linalg.norm(w)
        H[j + 1, j] = hn
        brk = hn <= 1e-14 * max(np.abs(H[: j + 2, j]).max(), 1.0)  # :125
        if not brk:
            V[j + 1] = w / hn
        for i in range(j):  # :130-133
            t = cs_[i] * H[i, j] + sn_[i] * H[i + 1, j]
            H[i + 1, j] = -np.conj(sn_[i]) * H[i, j] + cs_[i] * H[i + 1, j]
            H[i, j] = t
        a, hh = H[j, j], H[j + 1, j]
        rr = np.sqrt(np.abs(a) ** 2 + np.abs(hh) ** 2)  # :134-142
        if rr == 0.0:
            cs_[j], sn_[j] = 1.0, 0.0
        elif a == 0.0:
            cs_[j], sn_[j] = 0.0, np.conj(hh) / rr
        else:
            cs_[j] = np.abs(a) / rr
            sn_[j] = (a / np.abs(a)) * np.conj(hh) / rr
        H[j, j] = cs_[j] * a + sn_[j] * hh
        H[j + 1, j] = 0.0
        g[j + 1] = -np.conj(sn_[j]) * g[j]  # :145-146
        g[j] = cs_[j] * g[j]
        est = float(np.abs(g[j + 1]) / beta)
        hist.append(est)
        if est <= rtol or brk:  # :151-165
            x = solution(j)
            true_rel = float(np.linalg.norm(b - Aop(x)) / bnorm)
            conv = est <= rtol if left else true_rel <= rtol
            if conv or brk:
                rep = OReport(j + 1, conv, np.asarray(hist), true_rel, brk and not conv, x=x)
                rep.wall_seconds = time.perf_counter() - t0
                return rep
    x = solution(max_iter - 1)  # :167-175
    rep = OReport(max_iter, False, np.asarray(hist), float(np.linalg.norm(b - Aop(x)) / bnorm), x=x)
    rep.wall_seconds = time.perf_counter() - t0
    return rep


# --------------------------------------------------------------------------
# dense oracle (test_schwarz.py:22-42) for tiny instances
# --------------------------------------------------------------------------


def dense_preconditioner(kind, A, dec: ODecomposition, cs: OCoarse, weights_before_solve=False):
    """Explicit dense AS2/SAS2/SHS2 matrix — restates test_schwarz.py:22-42."""
    Ad = A.toarray()
    R0 = cs.r0.toarray().astype(Ad.dtype)
    C = R0.T @ np.linalg.solve(R0 @ Ad @ R0.T, R0)
    n = Ad.shape[0]
    loc = np.zeros_like(Ad)
    for s, w in zip(dec.index_sets, dec.weights):
        inv = np.linalg.inv(Ad[np.ix_(s, s)])
        if kind == "AS2":
            blk = inv
        elif weights_before_solve:
            blk = inv * w[None, :]
        else:
            blk = w[:, None] * inv
        loc[np.ix_(s, s)] += blk
    if kind in ("AS2", "SAS2"):
        return C + loc
    return C + loc @ (np.eye(n, dtype=Ad.dtype) - Ad @ C)
