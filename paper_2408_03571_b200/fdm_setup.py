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
    return _refine_eig(Ts, lam, U, np.diag(s))  # one Newton step (residual ~1e-13 -> ~1e-16)


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
    return _refine_eig(S, lam, U, Li.T)


def fold_bases(m: int):
    """Bases of the reflection-even / -odd subspaces of R^m (y -> m-1-y): Pe [m][he], Po [m][ho]."""
    he, ho = (m + 1) // 2, m // 2
    Pe = np.zeros((m, he))
    Po = np.zeros((m, ho))
    j = np.arange(ho)
    Pe[j, j] = Pe[m - 1 - j, j] = 1.0
    if he > ho:
        Pe[ho, ho] = 1.0
    Po[j, j] = 1.0
    Po[m - 1 - j, j] = -1.0
    return Pe, Po


def folded_pencil_eig(T0: np.ndarray, M0: np.ndarray):
    """T0 V = M0 V diag(lam), V^T M0 V = I for a reflection-symmetric pencil (J T0 J = T0,
    J M0 J = M0, J the y-reversal), solved on the even and odd subspaces separately: the
    modes come out exactly even (first he) or odd (last ho), so every product with V or
    V^T M0 folds to two half-size blocks (coarse.cu strip GEMMs)."""
    m = len(M0)
    J = np.arange(m)[::-1]
    if np.any(T0[np.ix_(J, J)] != T0) or np.any(M0[np.ix_(J, J)] != M0):
        raise ValueError("coarse y-pencil is not reflection symmetric")
    Pe, Po = fold_bases(m)
    lams, Vs = [], []
    for Pb in (Pe, Po):
        lb, Ub = _general_pencil_eig(Pb.T @ T0 @ Pb, Pb.T @ M0 @ Pb)
        lams.append(lb)
        Vs.append(Pb @ Ub)
    return np.concatenate(lams), np.concatenate(Vs, axis=1)


def fold_blocks(A: np.ndarray, kind: str) -> np.ndarray:
    """Packed half-size blocks of a mode/space matrix with reflection-parity structure:
    kind "left" (rows = modes [even; odd], columns = y: V^T M0, V^T) -> [A_e (he x he), A_o (ho x ho)]
    acting on Z_s = Z[y] + Z[m-1-y] (Z[h] alone for odd m) and Z_d = Z[y] - Z[m-1-y];
    kind "right" (rows = y, columns = modes: M0 V) -> [A_e, A_o] giving E[y] (y < he) and O[y]
    (y < ho), unfolded as out[y] = E + O, out[m-1-y] = E - O."""
    m = len(A)
    he, ho = (m + 1) // 2, m // 2
    if kind == "left":
        Ae, Ao = A[:he, :he], A[he:, :ho]
    else:
        Ae, Ao = A[:he, :he], A[:ho, he:]
    return np.concatenate([np.ascontiguousarray(Ae).ravel(), np.ascontiguousarray(Ao).ravel()])


def _refine_eig(S: np.ndarray, lam: np.ndarray, U: np.ndarray, back: np.ndarray):
    """One Newton step on S U = U diag(lam), U^T U = I for complex-symmetric S
    (the Ogita-Aishima update with the bilinear form in place of the inner product).

    LAPACK's non-symmetric eig leaves residuals ~1e-14 |S| that the Woodbury strip step
    amplifies to ~4e-12 in the coarse solve at m0 = 513; one step brings the residual to
    ~2e-15 (near-degenerate pairs, whose gap is below 1e-8 |S|, are left unmixed)."""
    R = np.eye(len(S)) - U.T @ U
    SU = U.T @ (S @ U)
    lt = np.diag(SU) / (1.0 - np.diag(R))
    gap = lt[None, :] - lt[:, None]
    tiny = np.abs(gap) < 1e-8 * np.abs(lt).max()
    E = np.where(tiny, 0.0, (SU + lt[None, :] * R) / np.where(tiny, 1.0, gap))
    np.fill_diagonal(E, np.diag(R) / 2)
    U = U + U @ E
    nrm = np.sqrt(np.einsum("ij,ij->j", U, U))
    U = U / nrm[None, :]
    return lt, back @ U


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


def _dst_pencil(L: int, h: float):
    """Exact eigen-pairs of tridiag(-1, 2, -1)/h^2 with W = I (every box with Dirichlet ends: all
    MP-1 boxes, the interior MP-2 boxes): lam_j = 4 sin^2(j pi / (2(L+1))) / h^2,
    V[i][j] = sqrt(2/(L+1)) sin(i j pi / (L+1)) (1-based), in long double -- LAPACK's eigenvalues
    carry an absolute error ~eps |T| that a near-resonant subdomain (lam_y + lam_x ~ k^2) turns
    into a ~1e-12 solve error."""
    ld = np.longdouble
    pi = ld("3.14159265358979323846264338327950288")
    j = np.arange(1, L + 1, dtype=ld)
    lam = (ld(4) / (ld(h) * ld(h))) * np.sin(j * pi / (2 * (L + 1))) ** 2
    V = np.sqrt(ld(2) / (L + 1)) * np.sin(np.outer(j, j) * pi / (L + 1))
    return lam.astype(np.float64), V.astype(np.float64)


def local_classes(grid: Grid, k: float, boxes) -> LocalClasses:
    """Eigen-pairs of every distinct 1-D box pencil (T[s:s+L, s:s+L], w[s:s+L])."""
    T, w = pencil_1d(grid, k)
    nu = grid.unknowns_per_dim
    h = grid.h
    keys, Vs, lams, cls = {}, [], [], []
    for s, L in boxes:
        key = (L, s == 0, s + L == nu)
        if key not in keys:
            Tb, wb = T[s : s + L, s : s + L], w[s : s + L]
            dirichlet_box = np.all(wb == 1.0) and not np.any(np.imag(Tb)) and \
                np.all(np.diag(Tb) == 2.0 / h**2) and np.all(np.diag(Tb, 1) == -1.0 / h**2)
            if dirichlet_box:
                lam, V = _dst_pencil(L, h)
                lam, V = lam.astype(T.dtype), V.astype(T.dtype)
            else:
                lam, V = _sym_pencil_eig(Tb, wb)
            keys[key] = len(Vs)
            Vs.append(V)
            lams.append(lam)
        cls.append(keys[key])
    # Every pair of 1-D classes occurs in some box (boxes are products of 1-D intervals).
    # A_i = T_y (x) W_x + W_y (x) T_x - k^2 W_y (x) W_x has the eigenvalues lam_y + lam_x - k^2;
    # where one is (numerically) zero the reference's splu hits a near-zero pivot and raises
    # SingularMatrixError (linalg.py:76-86, PIVOT_RTOL 1e-14 of max|A_i|): so does this setup.
    scale = float(np.abs(T).max() + k**2 * np.abs(w).max())
    for a in range(len(lams)):
        for b in range(len(lams)):
            den = np.abs(lams[a][:, None] + lams[b][None, :] - k**2)
            if den.min() <= 1e-14 * scale:
                raise SingularMatrixError(
                    f"subdomain matrix is singular: eigenvalue {den.min():.3e} (matrix scale {scale:.3e})")
    return LocalClasses(
        np.array([b[0] for b in boxes], np.int32),
        np.array([b[1] for b in boxes], np.int32),
        np.array(cls, np.int32),
        np.array([len(v) for v in Vs], np.int32),
        Vs,
        lams,
    )


@dataclass
class CoarseFast:
    """Setup of the fast coarse solver (one-time, host).

    A0 = T0(x)M0 + M0(x)T0 - k^2 M0(x)M0 (y (x) x).  Along x the 1-D pencil is
    split as T0 = T~ + L_T, M0 = M~ + L_M where (T~, M~) is diagonalised by a
    fast sine/cosine transform Q (T~ Q = W Q diag(lamT), M~ Q = W Q diag(lamM)):
    DST-I for Dirichlet (exact, L = 0), DCT-I for Sommerfeld (L_T, L_M live on
    the 2x2 corner blocks: the Bezier restriction drops its out-of-range taps
    instead of reflecting them, coarse.py:116-128).  B = T0(x)M~ + M0(x)T~ -
    k^2 M0(x)M~ is then x-transform + one pentadiagonal solve per x-mode; the
    corner corrections (4 strip columns) are removed by a Woodbury step whose
    capacitance matrix is block-diagonal (4x4) in the eigenbasis of the y-pencil.
    """

    m0: int
    transform: int          # 0: DST-I (Dirichlet), 1: DCT-I (Sommerfeld)
    scale: np.ndarray       # [m0] forward pre-scale sigma_a (Sommerfeld: qnorm/lamM[a]; Dirichlet: qnorm)
    lamT: np.ndarray        # [m0] eigenvalues of the ideal x-pencil (T~ Q = W Q diag(lamT))
    lamM: np.ndarray        # [m0]
    qn: float               # Dirichlet inverse-transform normalisation 2/(m0+1)
    k2: float
    shifts: np.ndarray      # [m0] s_a = lamT[a]/lamM[a] - k^2
    t0b: np.ndarray
    m0b: np.ndarray
    piv: np.ndarray         # band LU of T0 + s_a M0, layout [row][a]
    L: np.ndarray
    U: np.ndarray
    strip_x: np.ndarray     # [ns] x indices of the corrected columns (ns = 0 or 4)
    strip_q: np.ndarray     # [m0][ns] Q[strip_x[i], a]
    cap_left: np.ndarray    # [m0][m0]  V^T M0  (y-pencil eigenbasis, V^T M0 V = I)
    cap_right: np.ndarray   # [m0][m0]  M0 V
    cap_mode: np.ndarray    # [m0][ns][ns]  G_b (I + Gamma_b G_b)^{-1}
    # strip-space refinement (coarse.cu): the exact coupling on the strips and the
    # eigen-space approximation of (I + C_U G)^{-1} = I - H G used for the correction
    cap_vt: np.ndarray      # [m0][m0]  V^T
    cap_hg: np.ndarray      # [m0][ns][ns]  cap_mode_b Gamma_b
    strip_lt: np.ndarray    # [ns][ns]  (T0 - T~) on the strip columns
    strip_lm: np.ndarray    # [ns][ns]  (M0 - M~) on the strip columns


def _dense_from_bands(b: np.ndarray) -> np.ndarray:
    m = len(b)
    A = np.zeros((m, m), dtype=b.dtype)
    for d in range(-2, 3):
        i = np.arange(max(0, -d), min(m, m - d))
        A[i, i + d] = b[i, d + 2]
    return A


def coarse_pencil(grid: Grid, k: float):
    """T0 = P T P^T, M0 = P W P^T (pentadiagonal; A0 = T0(x)M0 + M0(x)T0 - k^2 M0(x)M0)."""
    T, w = pencil_1d(grid, k)
    P = bezier_1d(grid, 2)
    T0 = P @ T @ P.T
    M0 = P @ (w[:, None] * P.T)
    return 0.5 * (T0 + T0.T), 0.5 * (M0 + M0.T), P, T, w


def _transform_eigs(A: np.ndarray, dct: bool) -> np.ndarray:
    """diag(Q^{-1} W^{-1} A Q) of a pentadiagonal A in extended precision.

    The low modes of the stiffness pencil are tiny differences of O(1/h) entries: in
    fp64 they carry relative errors up to ~1e-11 (eps |T| / lambda_min), which the
    fast solve turns into a ~3e-12 solution error; long double (64-bit mantissa)
    sums bring them to the last fp64 bit."""
    m = len(A)
    ld = np.longdouble
    pi = ld("3.14159265358979323846264338327950288")
    I = np.arange(m, dtype=ld)
    if dct:
        Q = np.cos(np.outer(I, I) * (pi / (m - 1)))
        qn = np.full(m, ld(2) / (m - 1))
        qn[0] = qn[-1] = ld(1) / (m - 1)
    else:
        Q = np.sin(np.outer(I + 1, I + 1) * (pi / (m + 1)))
        qn = np.full(m, ld(2) / (m + 1))
    AQ = np.zeros((m, m), dtype=ld)
    for d in range(-2, 3):
        i = np.arange(max(0, -d), min(m, m - d))
        AQ[i] += A[i, i + d].astype(ld)[:, None] * Q[i + d]
    return ((Q * AQ).sum(axis=0) * qn).astype(np.float64)


def coarse_fast(grid: Grid, k: float) -> CoarseFast:
    """Fast-transform + Woodbury setup of A0^{-1} (replaces SuperLU of A0, coarse.py:154-167)."""
    T0, M0, P, T, w = coarse_pencil(grid, k)
    m = len(M0)
    I = np.arange(m)
    if grid.bc == "sommerfeld":
        Mx = m - 1
        Q = np.cos(np.pi * np.outer(I, I) / Mx)
        c = np.ones(m)
        c[0] = c[-1] = 2.0
        qnorm = 2.0 / (Mx * c)            # Q^{-1} W^{-1} = diag(qnorm) Q^T
        # Pi = P^T + E: the Bezier prolongation of the even (reflected) extension
        nu = grid.unknowns_per_dim
        Pi = P.T.copy()
        Pi[0, 1] += 1.0 / 8.0
        Pi[nu - 1, m - 2] += 1.0 / 8.0
        Tt = Pi.T @ T.real @ Pi
        Mt = Pi.T @ (w[:, None] * Pi)
        strip = np.array([0, 1, m - 2, m - 1], dtype=np.int32)
    else:
        Q = np.sin(np.pi * np.outer(I + 1, I + 1) / (m + 1))
        qnorm = np.full(m, 2.0 / (m + 1))
        Tt, Mt = T0.real, M0.real
        strip = np.zeros(0, dtype=np.int32)
    Qi = qnorm[:, None] * Q.T                 # Q^{-1} W^{-1}
    lamT = _transform_eigs(Tt.real, grid.bc == "sommerfeld")
    lamM = _transform_eigs(Mt.real, grid.bc == "sommerfeld")
    if np.any(lamM <= 0):
        raise SingularMatrixError("coarse mass pencil is not positive definite")
    shifts = lamT / lamM - k**2
    t0b, m0b = _bands(T0), _bands(M0)
    dt = T0.dtype
    if grid.bc == "sommerfeld":
        piv, L, U = band_lu(t0b, m0b.astype(dt), shifts.astype(dt))
        scale = qnorm / lamM
    else:  # the Dirichlet pencil is DST-diagonal in y as well: no band solves
        den = lamT[:, None] * lamM[None, :] + lamM[:, None] * lamT[None, :] - k**2 * np.outer(lamM, lamM)
        if np.any(np.abs(den) <= 1e-14 * np.abs(den).max()):
            raise SingularMatrixError("coarse Galerkin matrix is singular (k^2 at a coarse eigenvalue)")
        piv = np.zeros((0, 0), np.uint8)
        L = np.zeros((0, 0, 2), dt)
        U = np.zeros((0, 0, 5), dt)
        scale = qnorm.copy()
    ns = len(strip)
    strip_q = np.ascontiguousarray(Q[strip, :].T)  # [a][i]
    if ns:
        LT = (T0 - Tt)[np.ix_(strip, strip)]
        LM = (M0 - Mt)[np.ix_(strip, strip)]
        lam, V = folded_pencil_eig(T0, M0)
        den = lamM[None, :] * lam[:, None] + (lamT - k**2 * lamM)[None, :]  # [b][a]
        # Gamma_b[i][j] = sum_a Q[x_i,a] (Q^{-1}W^{-1})[a,x_j] / den[b,a]
        Gam = np.einsum("ai,aj,ba->bij", strip_q, Qi[:, strip], 1.0 / den)
        G = lam[:, None, None] * LM[None] + (LT - k**2 * LM)[None]
        K = np.eye(ns)[None] + Gam @ G
        cap_mode = G @ np.linalg.inv(K)
        cap_left, cap_right = V.T @ M0, M0 @ V
        cap_vt, cap_hg = V.T, cap_mode @ Gam
    else:
        cap_mode = cap_hg = np.zeros((m, 0, 0), dt)
        cap_left = cap_right = cap_vt = np.zeros((0, 0), dt)
        LT = LM = np.zeros((0, 0), dt)
    return CoarseFast(m, 1 if grid.bc == "sommerfeld" else 0, scale, lamT, lamM, float(qnorm[0]), float(k**2), shifts,
                      t0b,
                      m0b.astype(dt), piv,
                      L.astype(dt), U.astype(dt), strip, strip_q, cap_left.astype(dt), cap_right.astype(dt),
                      cap_mode.astype(dt), np.ascontiguousarray(cap_vt.astype(dt)), cap_hg.astype(dt),
                      np.asarray(LT, dt), np.asarray(LM, dt))


@dataclass
class CoarseDense:
    """Setup of the general coarse solver (FOCS any ratio, HOCS ratio 4/8/16; coarse.py:84-167).

    R0 = P (x) P with the banded 1-D P; A0 = T0(x)M0 + M0(x)T0 - k^2 M0(x)M0 (y (x) x) with
    T0 = P T P^T, M0 = P W P^T (Kronecker identity, exact for any P); the 1-D pencil
    T0 V = M0 V diag(lam), V^T M0 V = I gives A0^{-1} = (V(x)V) diag(1/(lam_y+lam_x-k^2)) (V(x)V)^T
    (coarse_dense.cu), refined on the device with the banded A0."""

    m0: int
    p_start: np.ndarray     # [m0]  int32
    p_taps: np.ndarray      # [m0][p_width]
    pt_start: np.ndarray    # [nu]  int32
    pt_taps: np.ndarray     # [nu][pt_width]
    bw: int                 # half-bandwidth of A0 along each axis
    a0_stencil: np.ndarray  # [m0*m0][(2bw+1)^2]  the reference's Galerkin matrix, row by row
    V: np.ndarray           # [m0][m0]
    invden: np.ndarray      # [m0][m0]


def _row_band(A: np.ndarray):
    """(start[r], taps[r][w]) of a banded dense matrix: row r's nonzeros lie in start..start+w-1."""
    nz = A != 0
    rows = A.shape[0]
    first = np.where(nz.any(axis=1), nz.argmax(axis=1), 0)
    last = np.where(nz.any(axis=1), A.shape[1] - 1 - nz[:, ::-1].argmax(axis=1), 0)
    w = int(max(1, (last - first).max() + 1))
    taps = np.zeros((rows, w))
    for r in range(rows):
        seg = A[r, first[r]: first[r] + w]
        taps[r, : len(seg)] = seg
    return first.astype(np.int32), taps


def _sym_band(A: np.ndarray, bw: int) -> np.ndarray:
    m = len(A)
    out = np.zeros((m, 2 * bw + 1), dtype=A.dtype)
    for d in range(-bw, bw + 1):
        i = np.arange(max(0, -d), min(m, m - d))
        out[i, d + bw] = A[i, i + d]
    return out


def assembled_matrix(grid: Grid, k: float):
    """The reference's CSR system matrix, built with the same sparse operations in the same
    order as helmdd discretization.py:128-188 (so its entries, and the Galerkin product below,
    carry the same rounding)."""
    import scipy.sparse as sp

    n, h = grid.n, grid.h
    if grid.bc == "dirichlet":
        m = n - 2
        ones = np.ones(m - 1)
        T = sp.diags([-ones, 2 * np.ones(m), -ones], [-1, 0, 1], format="csr") / h**2
        I = sp.identity(m, format="csr")
        A = sp.kron(T, I) + sp.kron(I, T) - k**2 * sp.identity(m * m)
    else:
        ones = np.ones(n - 1)
        T = sp.diags([-ones, 2 * np.ones(n), -ones], [-1, 0, 1], format="csr").astype(complex).tolil()
        T[0, 0] = 1.0
        T[n - 1, n - 1] = 1.0
        T = (T / h**2).tolil()
        T[0, 0] -= 1j * k / h
        T[n - 1, n - 1] -= 1j * k / h
        T = T.tocsr()
        w = np.ones(n)
        w[0] = w[-1] = 0.5
        W = sp.diags(w)
        A = sp.kron(T, W) + sp.kron(W, T) - k**2 * sp.kron(W, W)
    A = sp.csr_matrix(A)
    A.sort_indices()
    return A


def galerkin_stencil(grid: Grid, k: float, P: np.ndarray, bw: int) -> np.ndarray:
    """A0 = (B + B^T)/2 with B = R0 A R0^T, R0 = P (x) P, as helmdd coarse.py:136-139,154-165
    computes it, rearranged as a 2-D stencil [m0*m0][(2bw+1)^2]."""
    import scipy.sparse as sp

    A = assembled_matrix(grid, k)
    P1 = sp.csr_matrix(P)
    R0 = sp.kron(P1, P1, format="csr")
    R0.sort_indices()
    r0 = R0.astype(A.dtype)
    B = sp.csr_matrix(r0 @ A @ r0.T)
    a0 = ((B + B.T) * 0.5).tocoo()
    m = P.shape[0]
    wd = 2 * bw + 1
    iy, ix = np.divmod(a0.row, m)
    jy, jx = np.divmod(a0.col, m)
    dy, dx = jy - iy, jx - ix
    if np.abs(dy).max(initial=0) > bw or np.abs(dx).max(initial=0) > bw:
        raise ValueError("Galerkin matrix wider than the stencil half-width")
    st = np.zeros((m * m, wd * wd), dtype=A.dtype)
    st[a0.row, (dy + bw) * wd + dx + bw] = a0.data
    return st


def coarse_dense(grid: Grid, k: float, P: np.ndarray) -> CoarseDense:
    """Host setup of the general coarse solver for the 1-D restriction P (m0 x nu)."""
    T, w = pencil_1d(grid, k)
    T0 = P @ T @ P.T
    M0 = P @ (w[:, None] * P.T)
    T0, M0 = 0.5 * (T0 + T0.T), 0.5 * (M0 + M0.T)  # the symmetrisation of coarse.py:165
    m = len(M0)
    nzT = np.abs(T0) + np.abs(M0) > 0
    off = np.abs(np.subtract.outer(np.arange(m), np.arange(m)))
    bw = int(max(1, off[nzT].max()))
    lam, V = _general_pencil_eig(T0, M0)
    den = lam[:, None] + lam[None, :] - k**2
    scale = float(np.abs(T).max() + k**2 * np.abs(w).max())
    if np.abs(den).min() <= 1e-14 * scale:
        # the reference's splu of A0 hits a near-zero pivot here (linalg.py:76-86)
        raise SingularMatrixError(f"coarse Galerkin matrix is singular: eigenvalue {np.abs(den).min():.3e}")
    dt = T0.dtype
    ps, pt = _row_band(P)
    qs, qt = _row_band(np.ascontiguousarray(P.T))
    return CoarseDense(m, ps, pt, qs, qt, bw, galerkin_stencil(grid, k, P, bw),
                       np.ascontiguousarray(V.astype(dt)), np.ascontiguousarray((1.0 / den).astype(dt)))
