"""One-time host setup of the fast-diagonalisation (FDM) solvers.

The reference factorises every local matrix R_i A R_i^T (schwarz.py:55-59) and
the Galerkin matrix A0 = sym(R0 A R0^T) (coarse.py:154-167) with SuperLU.  Both
are Kronecker sums of 1-D pencils, so the B200 path only needs, once per
problem (SURVEY §8 hazard H8):

* local classes: for every distinct 1-D box pencil (T_box, W_box) the
  eigen-pairs  T V = W V diag(lambda)  with  V^T W V = I  (3 classes at most);
* coarse level: T0 = P T P^T, M0 = P W P^T (pentadiagonal), the eigen-pairs
  of (T0, M0) normalised V^T M0 V = I, and the pivoted band LU of
  T0 + (lambda_a - k^2) M0 for every a (partial FDM along x).

All of it is O(L^3) + O(m0^3) dense LAPACK on the host (seconds at n=2049);
the per-apply path never comes back here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla

from .discretization import Grid, bezier_1d, pencil_1d


class SingularMatrixError(ValueError):
    """A coarse or local pencil is (numerically) singular — helmdd linalg.py:18-24."""


def _sym_pencil_eig(T: np.ndarray, w: np.ndarray):
    """T V = diag(w) V diag(lam), V^T diag(w) V = I for (complex-)symmetric T, w > 0."""
    s = 1.0 / np.sqrt(w)
    Ts = s[:, None] * T * s[None, :]
    if not np.iscomplexobj(Ts) or not np.any(Ts.imag):
        lam, U = np.linalg.eigh(Ts.real)
        V = s[:, None] * U
        return lam.astype(T.dtype), V.astype(T.dtype)
    lam, U = np.linalg.eig(Ts)
    nrm = np.sqrt(np.einsum("ij,ij->j", U, U))  # complex-symmetric normalisation u^T u = 1
    U = U / nrm[None, :]
    return lam, s[:, None] * U


def _general_pencil_eig(T0: np.ndarray, M0: np.ndarray):
    """T0 V = M0 V diag(lam), V^T M0 V = I; M0 real SPD, T0 (complex) symmetric."""
    Lc = np.linalg.cholesky(M0)
    Li = sla.solve_triangular(Lc, np.eye(len(M0)), lower=True)
    S = Li @ T0 @ Li.T
    S = 0.5 * (S + S.T)
    if not np.iscomplexobj(S) or not np.any(S.imag):
        lam, U = np.linalg.eigh(S.real)
        return lam.astype(T0.dtype), (Li.T @ U).astype(T0.dtype)
    lam, U = np.linalg.eig(S)
    nrm = np.sqrt(np.einsum("ij,ij->j", U, U))
    U = U / nrm[None, :]
    return lam, Li.T @ U


def _bands(A: np.ndarray) -> np.ndarray:
    """[m][5] with out[i][d] = A[i][i+d-2] (zero outside)."""
    m = len(A)
    out = np.zeros((m, 5), dtype=A.dtype)
    for d in range(-2, 3):
        i = np.arange(max(0, -d), min(m, m - d))
        out[i, d + 2] = A[i, i + d]
    return out


def band_lu(t0b: np.ndarray, m0b: np.ndarray, shifts: np.ndarray):
    """Pivoted LU (partial pivoting, kl = ku = 2) of T0 + shift_a M0 for every a at once.

    Returns piv [m][na] (uint8, pivot row offset 0..2), L [m][na][2] multipliers
    and U [m][na][5] = {1/U_jj, U_j,j+1 .. U_j,j+4}; the layout [row][a] lets the
    device solve read the factors of consecutive systems with coalesced loads.
    """
    m, na = len(t0b), len(shifts)
    dt = np.result_type(t0b.dtype, m0b.dtype, shifts.dtype)
    B = t0b[None, :, :].astype(dt) + shifts[:, None, None] * m0b[None, :, :]  # (na, m, 5)
    piv = np.zeros((m, na), np.uint8)
    L = np.zeros((m, na, 2), dt)
    U = np.zeros((m, na, 5), dt)
    z = np.zeros((na, 1), dt)

    def orig_row(i):  # row i over columns i-2 .. i+2
        return B[:, i, :] if i < m else np.zeros((na, 5), dt)

    # active rows j, j+1, j+2 over columns j .. j+4
    R0 = np.concatenate([orig_row(0)[:, 2:], np.zeros((na, 2), dt)], axis=1)
    R1 = np.concatenate([orig_row(1)[:, 1:], z], axis=1) if m > 1 else np.zeros((na, 5), dt)
    R2 = orig_row(2).copy() if m > 2 else np.zeros((na, 5), dt)
    scale = np.abs(B).max(axis=(1, 2))
    idx = np.arange(na)
    for j in range(m):
        cand = np.stack([np.abs(R0[:, 0]), np.abs(R1[:, 0]), np.abs(R2[:, 0])], axis=1)
        if j + 1 >= m:
            cand[:, 1] = -1.0
        if j + 2 >= m:
            cand[:, 2] = -1.0
        pv = np.argmax(cand, axis=1)
        rows = np.stack([R0, R1, R2], axis=1)  # (na, 3, 5)
        top = rows[idx, pv].copy()
        rows[idx, pv] = rows[:, 0]
        rows[:, 0] = top
        R0, R1, R2 = rows[:, 0], rows[:, 1], rows[:, 2]
        d = R0[:, 0]
        if np.any(np.abs(d) <= 1e-14 * scale):
            raise SingularMatrixError("coarse band system is singular (k^2 at a coarse eigenvalue)")
        l1 = R1[:, 0] / d if j + 1 < m else np.zeros(na, dt)
        l2 = R2[:, 0] / d if j + 2 < m else np.zeros(na, dt)
        R1 = R1 - l1[:, None] * R0
        R2 = R2 - l2[:, None] * R0
        piv[j] = pv
        L[j, :, 0], L[j, :, 1] = l1, l2
        U[j, :, 0] = 1.0 / d
        U[j, :, 1:] = R0[:, 1:]
        R0 = np.concatenate([R1[:, 1:], z], axis=1)
        R1 = np.concatenate([R2[:, 1:], z], axis=1)
        R2 = orig_row(j + 3).copy()
    return piv, L, U


@dataclass
class LocalClasses:
    box_start: np.ndarray
    box_len: np.ndarray
    box_class: np.ndarray
    class_len: np.ndarray
    V: list
    lam: list


def local_classes(grid: Grid, k: float, boxes) -> LocalClasses:
    """Eigen-pairs of every distinct 1-D box pencil (T[s:s+L, s:s+L], w[s:s+L])."""
    T, w = pencil_1d(grid, k)
    nu = grid.unknowns_per_dim
    keys, Vs, lams, cls = {}, [], [], []
    for s, L in boxes:
        key = (L, s == 0, s + L == nu)
        if key not in keys:
            lam, V = _sym_pencil_eig(T[s : s + L, s : s + L], w[s : s + L])
            keys[key] = len(Vs)
            Vs.append(V)
            lams.append(lam)
        cls.append(keys[key])
    return LocalClasses(
        np.array([b[0] for b in boxes], np.int32),
        np.array([b[1] for b in boxes], np.int32),
        np.array(cls, np.int32),
        np.array([len(v) for v in Vs], np.int32),
        Vs,
        lams,
    )


@dataclass
class CoarseFDM:
    m0: int
    V: np.ndarray
    lam: np.ndarray
    t0b: np.ndarray
    m0b: np.ndarray
    piv: np.ndarray
    L: np.ndarray
    U: np.ndarray


def coarse_fdm(grid: Grid, k: float) -> CoarseFDM:
    """Partial-FDM data of A0 = T0(x)M0 + M0(x)T0 - k^2 M0(x)M0."""
    import scipy.sparse as sp

    nu, h = grid.unknowns_per_dim, grid.h
    e = np.ones(nu)
    dt = complex if grid.bc == "sommerfeld" else float
    d0 = np.full(nu, 2.0 / h**2, dtype=dt)
    w = np.ones(nu)
    if grid.bc == "sommerfeld":
        d0[0] = d0[-1] = 1.0 / h**2 - 1j * k / h
        w[0] = w[-1] = 0.5
    T = sp.diags([-e[1:] / h**2, d0, -e[1:] / h**2], [-1, 0, 1], format="csr")
    P = sp.csr_matrix(bezier_1d(grid, 2))
    T0 = (P @ T @ P.T).toarray()
    M0 = (P @ sp.diags(w) @ P.T).toarray()
    T0 = 0.5 * (T0 + T0.T)
    M0 = 0.5 * (M0 + M0.T)
    lam, V = _general_pencil_eig(T0, M0)
    t0b, m0b = _bands(T0), _bands(M0)
    shifts = (lam - k**2).astype(np.result_type(lam.dtype, T0.dtype))
    piv, L, U = band_lu(t0b, m0b, shifts)
    dt = T0.dtype
    return CoarseFDM(len(M0), V.astype(dt), lam.astype(dt), t0b, m0b.astype(dt), piv, L.astype(dt), U.astype(dt))
