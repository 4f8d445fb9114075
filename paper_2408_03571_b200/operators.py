"""Drop-in operators: the B200 replacements of ``A @ x`` and ``SchwarzPreconditioner.apply``.

Mirrors helmdd's public operator surface (``assemble(...).A``,
``SchwarzPreconditioner(kind, A, decomposition, coarse_space, ...)``,
``coarse_correct``) so the reference's own ``gmres`` — or this package's device
GMRES — can drive them.  Every application runs the sm_100a kernels of
``libhelmb200.so`` through its C ABI; there is no CPU compute path.

Vectors may be numpy arrays (copied host->device->host, so the unmodified
reference ``gmres`` can call us) or CUDA torch tensors (zero copy).  Both 1-D
``[N]`` and batched ``[batch, N]`` inputs are accepted.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .discretization import CoarseSpace, Decomposition, Grid, PROBLEMS, build_hocs, extend, partition
from .fdm_setup import CoarseDense, SingularMatrixError, coarse_dense, coarse_fast, fold_blocks, local_classes

__all__ = [
    "HelmholtzOperator",
    "HelmholtzProblem",
    "assemble",
    "galerkin",
    "coarse_correct",
    "SchwarzPreconditioner",
    "SingularMatrixError",
]


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


class _Vec:
    """Normalise an input vector to a contiguous CUDA tensor of the plan dtype."""

    def __init__(self, x, N: int, dtype: torch.dtype):
        self.numpy = isinstance(x, np.ndarray) or not isinstance(x, torch.Tensor)
        self.host_torch = isinstance(x, torch.Tensor) and not x.is_cuda
        if self.host_torch:  # host tensor (ideally pinned): async H2D, result copied back to the host
            if x.is_complex() and dtype == torch.float64:
                raise TypeError("complex input to a real (MP-1) operator is not supported on the device path")
            t = x.to(dtype).contiguous().to("cuda", non_blocking=True)
        elif self.numpy:
            arr = np.asarray(x)
            self.np_dtype = np.result_type(arr.dtype, np.complex128 if dtype == torch.complex128 else np.float64)
            if np.iscomplexobj(arr) and dtype == torch.float64:
                raise TypeError("complex input to a real (MP-1) operator is not supported on the device path")
            t = torch.from_numpy(np.ascontiguousarray(arr)).to(dtype)
            t = t.pin_memory().to("cuda", non_blocking=True) if t.numel() else t.to("cuda")
        else:
            if x.is_complex() and dtype == torch.float64:
                raise TypeError("complex input to a real (MP-1) operator is not supported on the device path")
            t = x.to(dtype).contiguous()
        if t.shape[-1] != N:
            raise ValueError(f"operator has dimension {N}, vector {t.shape[-1]}")
        if t.dim() not in (1, 2):
            raise ValueError("expected a vector [N] or a batch [batch, N]")
        self.t = t
        self.batch = 1 if t.dim() == 1 else t.shape[0]

    def empty_like(self, n=None):
        shape = self.t.shape if n is None else (*self.t.shape[:-1], n)
        return torch.empty(shape, dtype=self.t.dtype, device=self.t.device)

    def out(self, y: torch.Tensor, host_out=None):
        if self.numpy:
            return y.cpu().numpy()
        if self.host_torch:
            if host_out is None:
                host_out = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
            host_out.copy_(y, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return host_out
        return y


def _check_out(out, shape, dtype, device):
    """A caller-supplied result buffer: right dtype, shape, contiguity and device (CUDA out) or a
    host tensor of the same shape and dtype (pinned pipeline / host copy-back)."""
    if not isinstance(out, torch.Tensor):
        raise TypeError("out must be a torch tensor")
    if out.dtype != dtype:
        raise TypeError(f"out has dtype {out.dtype}, the operator computes in {dtype}")
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"out has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")
    if out.is_cuda and out.device != device:
        raise ValueError(f"out is on {out.device}, the input on {device}")


def _real_split(fn, x, N):
    """Apply a real-coefficient operator to a complex numpy vector by linearity (re, im)."""
    return fn(np.real(x)) + 1j * fn(np.imag(x))


class HelmholtzOperator:
    """Matrix-free 5-point Helmholtz operator A (helmdd discretization.py:157-191).

    ``A @ x`` launches K1.  It is immutable; ``plan`` is shared with the
    preconditioners built on it.
    """

    def __init__(self, grid: Grid, k: float, problem: str):
        self.grid, self.k, self.problem = grid, float(k), problem
        self.N = grid.num_unknowns
        self.dtype = np.complex128 if problem == "MP2" else np.float64
        self.torch_dtype = torch.complex128 if problem == "MP2" else torch.float64
        self.shape = (self.N, self.N)
        self._plan = None
        self._lock = threading.Lock()

    # the stencil only needs the grid part of a plan; it is created lazily so
    # that setting up an operator does not run the coarse eigen-solves
    def _stencil_plan(self, max_batch: int = 1):
        """The grid-only plan; its workspace is recreated when a caller needs more batch rows
        (unpreconditioned multi-RHS GMRES keeps nrhs Krylov bases in it)."""
        with self._lock:
            if self._plan is None or self._plan.max_batch < max_batch:
                self._plan = _Plan.create(self.grid, self.k, "SHS2", None, None, max_batch=max_batch)
            return self._plan

    def matvec(self, x):
        if isinstance(x, np.ndarray) and np.iscomplexobj(x) and self.dtype == np.float64:
            return _real_split(self.matvec, x, self.N)
        v = _Vec(x, self.N, self.torch_dtype)
        y = v.empty_like()
        plan = self._stencil_plan()
        _lib.check(plan.lib.helm_apply_A(plan.handle, _ptr(v.t), _ptr(y), v.batch, _stream()))
        return v.out(y)

    def __matmul__(self, x):
        if isinstance(x, np.ndarray) and x.ndim == 2 and x.shape[0] == self.N and x.shape[1] != self.N:
            return self.matvec(x.T).T  # scipy-style (N, k) columns
        return self.matvec(x)

    __call__ = matvec

    def tocsr(self):
        """Explicit CSR on the host (interop / tests only; never on the hot path)."""
        import scipy.sparse as sp

        from .discretization import pencil_1d

        T, w = pencil_1d(self.grid, self.k)
        T = sp.csr_matrix(T)
        W = sp.diags(w)
        A = sp.kron(T, W) + sp.kron(W, T) - self.k**2 * sp.kron(W, W)
        A = sp.csr_matrix(A)
        A.sort_indices()
        return A


@dataclass(frozen=True)
class HelmholtzProblem:
    grid: Grid
    k: float
    problem: str
    A: HelmholtzOperator
    f: np.ndarray


def assemble(grid: Grid, k: float, problem: str) -> HelmholtzProblem:
    """Problem setup (helmdd discretization.py:157-191): matrix-free A and the point load."""
    if problem not in PROBLEMS:
        raise ValueError(f"unknown problem {problem!r}, expected one of {PROBLEMS}")
    if k < 0:
        raise ValueError(f"wavenumber must be nonnegative, got {k}")
    expected = "dirichlet" if problem == "MP1" else "sommerfeld"
    if grid.bc != expected:
        raise ValueError(f"{problem} requires a {expected} grid, got {grid.bc!r}")
    # MP-2 accepts even n as the reference does (discretization.py:183-188: the load sits at the node
    # nearest the centre); the coarse spaces then need a ratio that divides n - 1 (coarse.py:78-79)
    if problem == "MP1" and grid.n % 2 == 0:
        raise ValueError("MP1 needs odd n so the source at (1/2, 1/2) is a grid node")
    A = HelmholtzOperator(grid, k, problem)
    f = np.zeros(grid.num_unknowns, dtype=A.dtype)
    c = (grid.n - 1) // 2
    f[grid.unknown_index(c, c)] = 1.0 / grid.h**2
    return HelmholtzProblem(grid, float(k), problem, A, f)


def _coarse_setup(cs, grid: Grid, k: float):
    """The coarse-solver setup for a coarse space: the fast transform + Woodbury solver for
    HOCS at ratio 2, the dense fast diagonalisation for every other space (coarse_dense.cu)."""
    kind, ratio = getattr(cs, "kind", "HOCS"), int(getattr(cs, "ratio", 2))
    if kind == "HOCS" and ratio == 2:
        return coarse_fast(grid, k)
    own = CoarseSpace(kind, grid, ratio)
    return coarse_dense(grid, k, own.restriction_1d())


def galerkin(cs: CoarseSpace, A) -> CoarseSpace:
    """Attach the coarse solver (replaces the SuperLU factorisation of A0, helmdd coarse.py:154-167)."""
    if cs.kind not in ("HOCS", "FOCS"):
        raise ValueError(f"unknown coarse space {cs.kind!r}")
    op = _as_operator(A, cs.grid)
    from dataclasses import replace

    if cs.kind == "HOCS" and cs.ratio == 2:
        # built where the plan is created: natively (helm_plan_create_problem) or by the host
        # setup of SchwarzPreconditioner(setup="host")
        return replace(cs, fdm=None)
    return replace(cs, fdm=_coarse_setup(cs, cs.grid, op.k))


class _Plan:
    """Owns a helm_plan + helm_workspace pair (C ABI handles)."""

    def __init__(self, lib, handle, ws, N, N0, keep):
        self.lib, self.handle, self.ws, self.N, self.N0 = lib, handle, ws, N, N0
        self._keep = keep
        self.lock = threading.Lock()

    @staticmethod
    def create(grid: Grid, k: float, kind: str, dec: Decomposition, cf, weights_before_solve=False,
               max_batch: int = 1, refine_steps: int = 0, strip_refine: int = 1):
        lib = _lib.load()
        cplx = grid.bc == "sommerfeld"
        dt = np.complex128 if cplx else np.float64
        i32 = lambda a: a.ctypes.data_as(_lib.c_int32_p)  # noqa: E731
        vp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
        d = _lib.HelmDesc()
        d.n, d.bc, d.is_complex = grid.n, (_lib.HELM_SOMMERFELD if cplx else _lib.HELM_DIRICHLET), int(cplx)
        d.kind, d.weights_before_solve = _lib.KINDS[kind], int(bool(weights_before_solve))
        d.ratio, d.k = 2, float(k)
        d.m0 = (grid.n - 3) // 2 if grid.bc == "dirichlet" else (grid.n + 1) // 2
        keep = {}
        if isinstance(cf, CoarseDense):  # general coarse space (coarse_dense.cu)
            d.ratio = (grid.n - 1) // (cf.m0 + (1 if grid.bc == "dirichlet" else -1))
            d.m0 = cf.m0
            for key, (v, t) in dict(ps=(cf.p_start, np.int32), pt=(cf.p_taps, np.float64),
                                    qs=(cf.pt_start, np.int32), qt=(cf.pt_taps, np.float64),
                                    st=(cf.a0_stencil, dt), V=(cf.V, dt), inv=(cf.invden, dt)).items():
                keep["cd_" + key] = np.ascontiguousarray(v, dtype=t)
            d.p_width, d.pt_width = cf.p_taps.shape[1], cf.pt_taps.shape[1]
            d.p_start, d.p_taps = i32(keep["cd_ps"]), vp(keep["cd_pt"])
            d.pt_start, d.pt_taps = i32(keep["cd_qs"]), vp(keep["cd_qt"])
            d.a0_bw, d.a0_stencil = cf.bw, vp(keep["cd_st"])
            d.coarse_V, d.coarse_invden = vp(keep["cd_V"]), vp(keep["cd_inv"])
            cf = None
        if dec is not None:  # subdomain FDM classes
            lc = local_classes(grid, k, dec.boxes)
            keep["classV"] = np.ascontiguousarray(np.concatenate([v.astype(dt).ravel() for v in lc.V]))
            keep["classL"] = np.ascontiguousarray(np.concatenate([l.astype(dt).ravel() for l in lc.lam]))
            for name in ("box_start", "box_len", "box_class", "class_len"):
                keep[name] = np.ascontiguousarray(getattr(lc, name), dtype=np.int32)
            d.p, d.overlap_layers = dec.p, dec.overlap_layers
            d.box_start, d.box_len = i32(keep["box_start"]), i32(keep["box_len"])
            d.box_class, d.class_len = i32(keep["box_class"]), i32(keep["class_len"])
            d.n_classes = len(lc.V)
            d.class_V, d.class_lambda = vp(keep["classV"]), vp(keep["classL"])
        if cf is not None:  # fast-transform + Woodbury coarse solver
            arrays = dict(scale=(cf.scale, np.float64), lamT=(cf.lamT, np.float64), lamM=(cf.lamM, np.float64),
                          t0b=(cf.t0b, dt), m0b=(cf.m0b, dt), piv=(cf.piv, np.uint8),
                          L=(cf.L, dt), U=(cf.U, dt), q=(cf.strip_q, np.float64), cm=(cf.cap_mode, dt), hg=(cf.cap_hg, dt),
                          lt=(cf.strip_lt, np.complex128), lm=(cf.strip_lm, np.complex128))
            if len(cf.strip_x):  # packed even/odd blocks (include/helmb200.h)
                arrays.update(cl=(fold_blocks(cf.cap_left, "left"), dt), cr=(fold_blocks(cf.cap_right, "right"), dt),
                              vt=(fold_blocks(cf.cap_vt, "left"), dt))
            for key, (v, t) in arrays.items():
                keep[key] = np.ascontiguousarray(v, dtype=t)
            d.coarse_scale = vp(keep["scale"])
            d.coarse_lamT, d.coarse_lamM, d.coarse_qn = vp(keep["lamT"]), vp(keep["lamM"]), cf.qn
            d.t0_band, d.m0_band = vp(keep["t0b"]), vp(keep["m0b"])
            if cplx:
                d.band_piv = keep["piv"].ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
                d.band_l, d.band_u = vp(keep["L"]), vp(keep["U"])
            d.n_strip = len(cf.strip_x)
            if d.n_strip:
                d.strip_q, d.cap_left, d.cap_right = vp(keep["q"]), vp(keep["cl"]), vp(keep["cr"])
                d.cap_mode = vp(keep["cm"])
                d.cap_vt, d.cap_hg = vp(keep["vt"]), vp(keep["hg"])
                d.strip_lt, d.strip_lm = vp(keep["lt"]), vp(keep["lm"])
                d.strip_refine = int(strip_refine)
        d.refine_steps = int(refine_steps)
        h = ctypes.c_void_p()
        _lib.check(lib.helm_plan_create(ctypes.byref(d), ctypes.byref(h)))
        ws = ctypes.c_void_p()
        try:
            _lib.check(lib.helm_workspace_create(h, int(max_batch), ctypes.byref(ws)))
        except Exception:
            lib.helm_plan_destroy(h)
            raise
        plan = _Plan(lib, h, ws, lib.helm_plan_num_unknowns(h), lib.helm_plan_num_coarse(h), None)
        plan.max_batch = int(max_batch)
        return plan

    @staticmethod
    def create_native(grid: Grid, k: float, kind: str, dec: Decomposition, weights_before_solve=False,
                      max_batch: int = 1, refine_steps: int = 0, strip_refine: int = 1):
        """The plan from the problem parameters alone: helm_plan_create_problem builds the box
        classes, eigen-pairs (cuSOLVER), transform eigenvalues, band LU and Woodbury data natively
        (include/helmb200.h).  HOCS ratio 2 only."""
        lib = _lib.load()
        pr = _lib.HelmProblem()
        pr.n, pr.bc = grid.n, (_lib.HELM_SOMMERFELD if grid.bc == "sommerfeld" else _lib.HELM_DIRICHLET)
        pr.kind, pr.weights_before_solve = _lib.KINDS[kind], int(bool(weights_before_solve))
        pr.p, pr.overlap_layers, pr.coarse_kind, pr.ratio, pr.k = dec.p, dec.overlap_layers, 0, 2, float(k)
        pr.strip_refine, pr.refine_steps = int(strip_refine), int(refine_steps)
        h = ctypes.c_void_p()
        status = lib.helm_plan_create_problem(ctypes.byref(pr), ctypes.byref(h))
        if status != 0:
            msg = lib.helm_last_error().decode(errors="replace")
            if "singular" in msg:
                raise SingularMatrixError(msg)
            raise _lib.HelmError(msg)
        ws = ctypes.c_void_p()
        try:
            _lib.check(lib.helm_workspace_create(h, int(max_batch), ctypes.byref(ws)))
        except Exception:
            lib.helm_plan_destroy(h)
            raise
        plan = _Plan(lib, h, ws, lib.helm_plan_num_unknowns(h), lib.helm_plan_num_coarse(h), None)
        plan.max_batch = int(max_batch)
        return plan

    def __del__(self):
        try:
            if self.ws:
                self.lib.helm_workspace_destroy(self.ws)
            if self.handle:
                self.lib.helm_plan_destroy(self.handle)
        except Exception:
            pass


def _as_operator(A, grid: Grid) -> HelmholtzOperator:
    """Accept our operator, or a reference CSR matrix after a structure guard."""
    if isinstance(A, HelmholtzOperator):
        return A
    import scipy.sparse as sp

    if sp.issparse(A):
        problem = "MP1" if grid.bc == "dirichlet" else "MP2"
        if A.shape != (grid.num_unknowns, grid.num_unknowns):
            raise ValueError("matrix size does not match the decomposition's grid")
        # recover k from an interior diagonal entry: 4/h^2 - k^2
        c = (grid.unknowns_per_dim // 2) * (grid.unknowns_per_dim + 1)
        k2 = 4.0 / grid.h**2 - float(np.real(A[c, c]))
        op = HelmholtzOperator(grid, float(np.sqrt(max(k2, 0.0))), problem)
        ref = op.tocsr()
        if abs(ref - A).max() > 1e-12 * abs(A).max():
            raise ValueError("A is not the constant-k 5-point Helmholtz operator of this grid")
        return op
    raise TypeError("A must be a HelmholtzOperator or the reference's assembled CSR matrix")


def _grid_of(obj) -> Grid:
    g = obj.grid
    return g if isinstance(g, Grid) else Grid(g.n, g.bc)


class SchwarzPreconditioner:
    """Two-level Schwarz M^{-1} (AS2 / SAS2 / SHS2) on the B200 — helmdd schwarz.py:31-103.

    Immutable after construction; ``apply`` serialises on an internal lock
    because the device workspace is shared (the reference's concurrent-read
    contract holds for callers).  ``decomposition`` / ``coarse_space`` may be
    this package's descriptors or the reference's objects (duck-typed).
    """

    KINDS = ("AS2", "SAS2", "SHS2")

    def __init__(self, kind, A, decomposition, coarse_space, weights_before_solve=False,
                 local_factorizations=None, max_batch: int = 1, refine_steps=None, strip_refine: int = 1,
                 setup: str = None):
        """``setup``: "host" (numpy/LAPACK setup in fdm_setup.py, then helm_plan_create) or "native"
        (helm_plan_create_problem: the library builds everything from the problem parameters; HOCS
        ratio 2).  Default: HELM_SETUP or "native" where it applies."""
        if kind not in self.KINDS:
            raise ValueError(f"unknown preconditioner {kind!r}, expected one of {self.KINDS}")
        grid = _grid_of(decomposition)
        if A.shape[0] != grid.num_unknowns:
            raise ValueError("matrix size does not match the decomposition's grid")
        self.kind = kind
        self.A = _as_operator(A, grid)
        self.decomposition = Decomposition(grid, decomposition.p, decomposition.overlap_layers)
        ckind, ratio = getattr(coarse_space, "kind", "HOCS"), int(getattr(coarse_space, "ratio", 2))
        if ckind not in ("HOCS", "FOCS"):
            raise ValueError(f"unknown coarse space {ckind!r}")
        import os

        setup = setup or os.environ.get("HELM_SETUP", "native")
        if setup not in ("host", "native"):
            raise ValueError(f"setup must be 'host' or 'native', got {setup!r}")
        native = setup == "native" and ckind == "HOCS" and ratio == 2
        self.weights_before_solve = bool(weights_before_solve)
        self.max_batch = int(max_batch)
        self.setup = "native" if native else "host"
        if native:
            self.coarse_space = CoarseSpace(ckind, grid, ratio, None)
            self.plan = _Plan.create_native(grid, self.A.k, kind, self.decomposition, weights_before_solve,
                                            max_batch=max_batch, refine_steps=refine_steps or 0,
                                            strip_refine=strip_refine)
            self.N, self.N0 = self.plan.N, self.plan.N0
            return
        cf = getattr(coarse_space, "fdm", None)
        if cf is None:
            cf = _coarse_setup(coarse_space, grid, self.A.k)
        self.coarse_space = CoarseSpace(ckind, grid, ratio, cf)
        if refine_steps is None:  # the dense coarse solve is refined twice (coarse_dense.cu)
            refine_steps = 2 if isinstance(cf, CoarseDense) else 0
        self.plan = _Plan.create(grid, self.A.k, kind, self.decomposition, cf, weights_before_solve,
                                 max_batch=max_batch, refine_steps=refine_steps, strip_refine=strip_refine)
        self.N = self.plan.N
        self.N0 = self.plan.N0

    # -- the individual operators (for parity tests and benchmarks) ---------
    def _run(self, fn, x, out_len=None, in_len=None, out=None):
        v = _Vec(x, in_len or self.N, self.A.torch_dtype)
        if v.batch > self.max_batch:
            raise ValueError(f"batch {v.batch} exceeds max_batch {self.max_batch}")
        shape = (*v.t.shape[:-1], out_len or self.N)
        if out is not None:  # the kernels write through the raw pointer: the buffer must match exactly
            _check_out(out, shape, self.A.torch_dtype, v.t.device)
        y = out if (out is not None and out.is_cuda) else v.empty_like(out_len or self.N)
        with self.plan.lock:
            _lib.check(fn(v.t, y, v.batch))
        return v.out(y, host_out=out if (out is not None and not out.is_cuda) else None)

    def apply(self, x, out=None):
        """y = M^{-1} x.  ``out``: optional preallocated result (CUDA tensor, or pinned host
        tensor when ``x`` is a host tensor)."""
        if isinstance(x, np.ndarray) and np.iscomplexobj(x) and self.A.dtype == np.float64:
            return _real_split(self.apply, x, self.N)
        p = self.plan
        if (isinstance(x, torch.Tensor) and not x.is_cuda and x.is_pinned() and x.dim() == 2 and x.is_contiguous()
                and x.dtype == self.A.torch_dtype and x.shape[0] > self.PIPE_CHUNK and x.shape[1] == self.N
                and out is not None and not out.is_cuda and out.is_pinned() and out.shape == x.shape):
            return self._apply_pipelined(x, out)
        return self._run(lambda a, b, n: p.lib.helm_apply_M(p.handle, p.ws, _ptr(a), _ptr(b), n, _stream()), x,
                         out=out)

    __call__ = apply

    # vectors per pipeline chunk; smaller chunks shorten the unoverlapped first H2D and last D2H
    # (config 5, 32 vectors: 2 -> 627, 4 -> 619, 8 -> 570, 16 -> 494 applies/s, tools/e2e_chunk.py)
    PIPE_CHUNK = 2

    def _apply_pipelined(self, xh: torch.Tensor, yh: torch.Tensor):
        """Host batch -> host batch with the PCIe copies overlapped with the kernels.

        The batch is cut into chunks of PIPE_CHUNK vectors; chunk i+1 is copied
        host->device on one stream while chunk i runs through the kernels on the current
        stream and chunk i-1 is copied device->host on a third, with two device buffers
        per direction (events order the reuse).  Returns when ``yh`` holds the result."""
        p = self.plan
        cb = self.PIPE_CHUNK
        comp = torch.cuda.current_stream()
        st = getattr(self, "_pipe", None)
        if st is None or st["bufs_in"][0].shape[0] != cb:
            mk = lambda: torch.empty((cb, self.N), dtype=self.A.torch_dtype, device="cuda")  # noqa: E731
            st = dict(s_in=torch.cuda.Stream(), s_out=torch.cuda.Stream(), bufs_in=[mk(), mk()],
                      bufs_out=[mk(), mk()])
            self._pipe = st
        s_in, s_out = st["s_in"], st["s_out"]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_comp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]
        nb = xh.shape[0]
        with self.plan.lock:
            for i, lo in enumerate(range(0, nb, cb)):
                hi, k = min(nb, lo + cb), i % 2
                bi, bo = st["bufs_in"][k][: hi - lo], st["bufs_out"][k][: hi - lo]
                if used[k]:
                    s_in.wait_event(ev_comp[k])  # the kernels of chunk i-2 have consumed bufs_in[k]
                with torch.cuda.stream(s_in):
                    bi.copy_(xh[lo:hi], non_blocking=True)
                    ev_in[k].record(s_in)
                comp.wait_event(ev_in[k])
                if used[k]:
                    comp.wait_event(ev_out[k])  # chunk i-2's result has left bufs_out[k]
                _lib.check(p.lib.helm_apply_M(p.handle, p.ws, _ptr(bi), _ptr(bo), hi - lo,
                                              ctypes.c_void_p(comp.cuda_stream)))
                ev_comp[k].record(comp)
                s_out.wait_event(ev_comp[k])
                with torch.cuda.stream(s_out):
                    yh[lo:hi].copy_(bo, non_blocking=True)
                    ev_out[k].record(s_out)
                used[k] = True
            s_out.synchronize()
        return yh

    def restrict(self, x):
        p = self.plan
        return self._run(lambda a, b, n: p.lib.helm_restrict(p.handle, _ptr(a), _ptr(b), n, _stream()), x,
                         self.N0)

    def prolong(self, c):
        p = self.plan
        return self._run(lambda a, b, n: p.lib.helm_prolong(p.handle, _ptr(a), _ptr(b), n, _stream()), c,
                         self.N, self.N0)

    def coarse_solve(self, c):
        p = self.plan
        return self._run(lambda a, b, n: p.lib.helm_coarse_solve(p.handle, p.ws, _ptr(a), _ptr(b), n, _stream()),
                         c, self.N0, self.N0)

    def coarse_correct(self, x):
        p = self.plan
        return self._run(lambda a, b, n: p.lib.helm_coarse_correct(p.handle, p.ws, _ptr(a), _ptr(b), n, _stream()),
                         x)

    def local_sum(self, x, weighted=True, base=None):
        """y = base + sum_i R_i^T [D_i] A_i^{-1} [D_i] R_i x  (helmdd schwarz.py:64-74)."""
        p = self.plan
        bt = None
        if base is not None:
            bt = _Vec(base, self.N, self.A.torch_dtype).t
            xb = 1 if (not hasattr(x, "shape") or len(x.shape) == 1) else x.shape[0]
            bb = 1 if bt.dim() == 1 else bt.shape[0]
            if bb != xb:  # the kernel reads base + b*N for every batch row b
                raise ValueError(f"base has {bb} rows, x has {xb}")
        return self._run(
            lambda a, b, n: p.lib.helm_local_sum(p.handle, p.ws, _ptr(a), _ptr(bt) if bt is not None else None,
                                                 _ptr(b), int(weighted), n, _stream()), x)


def coarse_correct(M: SchwarzPreconditioner, r):
    """R0^T A0^{-1} R0 r (helmdd coarse.py:170-174) on the preconditioner's plan."""
    return M.coarse_correct(r)
