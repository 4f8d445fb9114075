"""Device GMRES — drop-in for helmdd ``gmres(A, M_inv, b, cfg) -> SolveReport`` (gmres.py:29-177).

The whole loop runs in ``helm_gmres`` (libhelmb200.so): Krylov basis, Hessenberg
matrix, Givens rotations and residual estimates live in HBM; the host reads one
estimate per iteration to decide termination, exactly where the reference's
Python loop tests ``estimate <= rtol`` (gmres.py:151).  Stopping semantics are
the reference's: right preconditioning confirms on the true residual
``||b - A x|| / ||b||`` before declaring convergence; left stops on the
estimate; breakdown ``h_{j+1,j} <= 1e-14 max(max|H[:j+2,j]|, 1)`` terminates.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .operators import HelmholtzOperator, SchwarzPreconditioner, _as_operator, _ptr, _stream, _Vec

__all__ = ["GmresConfig", "SolveReport", "gmres", "gmres_multi"]


@dataclass(frozen=True)
class GmresConfig:
    """helmdd gmres.py:29-41 (defaults rtol 1e-7, max_iter 100, side 'right')."""

    rtol: float = 1e-7
    max_iter: int = 100
    side: str = "right"

    def __post_init__(self):
        if self.rtol <= 0:
            raise ValueError(f"relative tolerance must be positive, got {self.rtol}")
        if self.max_iter < 1:
            raise ValueError(f"iteration cap must be at least 1, got {self.max_iter}")
        if self.side not in ("left", "right"):
            raise ValueError(f"preconditioning side must be 'left' or 'right', got {self.side!r}")


@dataclass
class SolveReport:
    """helmdd gmres.py:44-54."""

    iterations: int
    converged: bool
    residual_history: np.ndarray
    final_residual: float
    breakdown: bool = False
    wall_seconds: float = field(default=0.0)
    x: object = None
    reorth_iterations: int = 0  # iterations whose conditional re-orthogonalisation ran (device detail)


def _resolve(A, M_inv):
    """(operator, plan, use_precond).  The device loop applies the plan's own stencil, so a
    given ``A`` must BE that operator (gmres.py:57-62 treats A and M_inv independently): the
    preconditioner's operator, or one with the same grid, k and problem, or the reference's
    CSR of it (structure guard)."""
    if M_inv is not None and not isinstance(M_inv, SchwarzPreconditioner):
        raise TypeError("device GMRES needs M_inv to be a SchwarzPreconditioner of this package (or None)")
    if M_inv is None:
        if A is None:
            raise TypeError("A is required")
        op = A if isinstance(A, HelmholtzOperator) else None
        if op is None:
            raise TypeError("with M_inv=None, A must be a HelmholtzOperator")
        return op, op._stencil_plan(), 0
    op = M_inv.A
    if A is not None and A is not op:
        given = _as_operator(A, op.grid)  # CSR: structure guard (k recovered, entries compared)
        if (given.grid.n, given.grid.bc, given.problem) != (op.grid.n, op.grid.bc, op.problem) or \
                abs(given.k - op.k) > 1e-12 * max(1.0, op.k):
            raise ValueError("A differs from the operator the preconditioner was built on "
                             f"(k {given.k} vs {op.k}, n {given.grid.n} vs {op.grid.n}, {given.problem} vs {op.problem})")
    return op, M_inv.plan, 1


def gmres(A, M_inv, b, cfg: GmresConfig = GmresConfig()) -> SolveReport:
    """Solve A x = b with the B200 preconditioner ``M_inv`` (a SchwarzPreconditioner or None)."""
    op, plan, use_precond = _resolve(A, M_inv)
    v = _Vec(b, op.N, op.torch_dtype)
    if v.batch != 1 or v.t.dim() != 1:
        raise ValueError("gmres solves one right-hand side")
    x = torch.empty_like(v.t)
    hist = np.zeros(cfg.max_iter + 1)
    rep = _lib.HelmGmresReport()
    with plan.lock:
        status = plan.lib.helm_gmres(
            plan.handle, plan.ws, _ptr(v.t), _ptr(x), float(cfg.rtol), int(cfg.max_iter),
            1 if cfg.side == "left" else 0, use_precond,
            hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(rep), _stream(),
        )
    if status != 0:
        msg = plan.lib.helm_last_error().decode(errors="replace")
        if "nonzero" in msg:
            raise ValueError(msg)
        raise _lib.HelmError(msg)
    return SolveReport(
        iterations=rep.iterations,
        converged=bool(rep.converged),
        residual_history=hist[: rep.iterations + 1].copy(),
        final_residual=float(rep.final_residual),
        breakdown=bool(rep.breakdown),
        wall_seconds=float(rep.wall_seconds),
        x=v.out(x),
        reorth_iterations=int(rep.reorth),
    )


def gmres_multi(A, M_inv, B, cfg: GmresConfig = GmresConfig()) -> list:
    """Solve A x_r = b_r for the rows b_r of ``B`` ([nrhs, N]) with one GMRES per right-hand
    side (the reference's loop, gmres.py:65-177, for each) sharing every application of A and
    M^{-1} (``helm_gmres_multi``: the batched kernels at batch nrhs).  ``M_inv`` needs
    ``max_batch >= nrhs``.  Returns one SolveReport per row; ``wall_seconds`` is the whole
    call's.  Not in the reference."""
    op, plan, use_precond = _resolve(A, M_inv)
    v = _Vec(B, op.N, op.torch_dtype)
    if v.t.dim() != 2:
        raise ValueError("gmres_multi expects right-hand sides as rows of a [nrhs, N] array")
    nrhs = v.batch
    if M_inv is None:
        plan = op._stencil_plan(max_batch=nrhs)
    if M_inv is not None and nrhs > M_inv.max_batch:
        raise ValueError(f"{nrhs} right-hand sides exceed the preconditioner's max_batch {M_inv.max_batch}")
    x = torch.empty_like(v.t)
    hist = np.zeros((nrhs, cfg.max_iter + 1))
    reps = (_lib.HelmGmresReport * nrhs)()
    with plan.lock:
        status = plan.lib.helm_gmres_multi(
            plan.handle, plan.ws, _ptr(v.t), _ptr(x), nrhs, float(cfg.rtol), int(cfg.max_iter),
            1 if cfg.side == "left" else 0, use_precond,
            hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), reps, _stream(),
        )
    if status != 0:
        msg = plan.lib.helm_last_error().decode(errors="replace")
        if "nonzero" in msg:
            raise ValueError(msg)
        raise _lib.HelmError(msg)
    xs = v.out(x)
    return [
        SolveReport(
            iterations=reps[q].iterations,
            converged=bool(reps[q].converged),
            residual_history=hist[q, : reps[q].iterations + 1].copy(),
            final_residual=float(reps[q].final_residual),
            breakdown=bool(reps[q].breakdown),
            wall_seconds=float(reps[q].wall_seconds),
            x=xs[q],
        )
        for q in range(nrhs)
    ]
