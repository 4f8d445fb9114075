"""numpy emulation of the device FDM algorithms (test helper, CPU only).

Re-implements, statement for statement, what the CUDA kernels K4 (local FDM)
and K5 (fast x-transform + band solves + Woodbury strip correction + iterative refinement) compute, so the
host setup (eigen-pairs, band LU) can be validated against the oracle's
SuperLU solves without a GPU.
"""

from __future__ import annotations

import numpy as np


def band_solve(piv, L, U, G):
    """Solve column systems exactly like band_solve_kernel (G: [m][na], in place copy)."""
    m, na = G.shape
    out = np.array(G, dtype=np.result_type(G.dtype, L.dtype))
    r0 = out[0].copy()
    r1 = out[1].copy() if m > 1 else np.zeros(na, out.dtype)
    r2 = out[2].copy() if m > 2 else np.zeros(na, out.dtype)
    idx = np.arange(na)
    for j in range(m):
        rows = np.stack([r0, r1, r2])
        pv = piv[j]
        top = rows[pv, idx].copy()
        rows[pv, idx] = rows[0]
        rows[0] = top
        r0, r1, r2 = rows
        r1 = r1 - L[j, :, 0] * r0
        r2 = r2 - L[j, :, 1] * r0
        out[j] = r0
        r0, r1 = r1, r2
        r2 = out[j + 3].copy() if j + 3 < m else np.zeros(na, out.dtype)
    xs = [np.zeros(na, out.dtype) for _ in range(4)]
    for j in range(m - 1, -1, -1):
        u = U[j]
        v = out[j] - u[:, 1] * xs[0] - u[:, 2] * xs[1] - u[:, 3] * xs[2] - u[:, 4] * xs[3]
        v = v * u[:, 0]
        out[j] = v
        xs = [v] + xs[:3]
    return out


def a0_apply(cf, k, Y):
    """A0 Y = T0 Y M0^T + M0 Y T0^T - k^2 M0 Y M0^T from the bands."""
    m = cf.m0

    def dense(b):
        A = np.zeros((m, m), dtype=b.dtype)
        for d in range(-2, 3):
            i = np.arange(max(0, -d), min(m, m - d))
            A[i, i + d] = b[i, d + 2]
        return A

    T0, M0 = dense(cf.t0b), dense(cf.m0b)
    return T0 @ Y @ M0.T + M0 @ Y @ T0.T - k**2 * (M0 @ Y @ M0.T)


def x_transform(cf, X):
    """Raw DST-I / DCT-I sums along x (rows of X): out[y, a] = sum_J Q[J, a] X[y, J]."""
    m = cf.m0
    I = np.arange(m)
    if cf.transform == 1:
        Q = np.cos(np.pi * np.outer(I, I) / (m - 1))
    else:
        Q = np.sin(np.pi * np.outer(I + 1, I + 1) / (m + 1))
    return X @ Q


def _dense_bands(b):
    m = len(b)
    A = np.zeros((m, m), dtype=b.dtype)
    for d in range(-2, 3):
        i = np.arange(max(0, -d), min(m, m - d))
        A[i, i + d] = b[i, d + 2]
    return A


def strip_coupling(cf, YS):
    """C_U y_S = (A0 - B) restricted to the strip columns (strip_rho_kernel)."""
    T0, M0 = _dense_bands(cf.t0b), _dense_bands(cf.m0b)
    return T0 @ YS @ cf.strip_lm.T + M0 @ YS @ (cf.strip_lt - cf.k2 * cf.strip_lm).T


def fast_solve(cf, R, strip_refine=0):
    """One pass of the device coarse solve (coarse.cu): x-transform, band solves + Woodbury strip
    step (Sommerfeld) or the separable 2-D DST scaling (Dirichlet), inverse transform.
    strip_refine: Newton steps on the strip coupling (Sommerfeld), each one more band pass."""
    Fh = x_transform(cf, R) * cf.scale[None, :]
    if cf.transform == 0:
        lT, lM = cf.lamT, cf.lamM
        den = lT[:, None] * lM[None, :] + lM[:, None] * lT[None, :] - cf.k2 * np.outer(lM, lM)  # [ky][kx]
        G = x_transform(cf, Fh.T).T * cf.qn / den
        return x_transform(cf, x_transform(cf, G.T).T)
    if len(cf.strip_x):
        Y0h = band_solve(cf.piv, cf.L, cf.U, Fh)
        Y0S = Y0h @ cf.strip_q                          # strip columns of B^{-1} R
        yh = cf.cap_left @ Y0S                          # y-eigen coordinates
        ch = np.einsum("bij,bj->bi", cf.cap_mode, yh)   # per-mode 4x4
        cS = cf.cap_right @ ch
        Yh = band_solve(cf.piv, cf.L, cf.U, Fh - (cS @ cf.strip_q.T) * cf.scale[None, :])
        for _ in range(strip_refine):
            # true residual on the strips, rho = c - C_U y_S (exact: y_S from the band pass)
            rho = cS - strip_coupling(cf, Yh @ cf.strip_q)
            t = np.einsum("bij,bj->bi", cf.cap_hg, cf.cap_vt @ rho)
            w = cf.cap_right @ t - rho               # -(I - H G) rho
            Yh = Yh + band_solve(cf.piv, cf.L, cf.U, -(w @ cf.strip_q.T) * cf.scale[None, :])
            cS = cS + w
        return x_transform(cf, Yh)
    Yh = band_solve(cf.piv, cf.L, cf.U, Fh)
    return x_transform(cf, Yh)


def coarse_solve(cf, k, c, refine=0, strip_refine=1):
    m = cf.m0
    C = c.reshape(m, m)
    Y = fast_solve(cf, C, strip_refine)
    for _ in range(refine):
        Y = Y + fast_solve(cf, C - a0_apply(cf, k, Y), strip_refine)
    return Y.ravel()


def local_sum(dec, lc, k, x, weighted=True):
    nu = dec.grid.unknowns_per_dim
    X = x.reshape(nu, nu)
    out = np.zeros_like(X, dtype=np.result_type(X.dtype, lc.V[0].dtype))
    mult = dec.multiplicity_1d
    for ay in range(dec.p):
        for ax in range(dec.p):
            ys, yl = lc.box_start[ay], lc.box_len[ay]
            xs, xl = lc.box_start[ax], lc.box_len[ax]
            Vy, ly = lc.V[lc.box_class[ay]], lc.lam[lc.box_class[ay]]
            Vx, lx = lc.V[lc.box_class[ax]], lc.lam[lc.box_class[ax]]
            Xi = X[ys : ys + yl, xs : xs + xl]
            Y = (Vy.T @ Xi @ Vx) / (ly[:, None] + lx[None, :] - k**2)
            Y = Vy @ Y @ Vx.T
            if weighted:
                Y = Y / np.outer(mult[ys : ys + yl], mult[xs : xs + xl])
            out[ys : ys + yl, xs : xs + xl] += Y
    return out.ravel()
