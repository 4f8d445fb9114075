"""Grid, problem and subdomain descriptors — the host-side mirror of the reference's
setup objects (``discretization.py``, ``decomposition.py``, ``coarse.py`` of helmdd).

Nothing here assembles a sparse matrix on the hot path: ``assemble`` returns a
matrix-free :class:`HelmholtzOperator` whose ``@`` runs the sm_100a stencil
kernel (K1).  ``partition``/``extend`` only describe the boxes; their index
sets and weights are materialised lazily for callers that ask for them.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

PROBLEMS = ("MP1", "MP2")


@dataclass(frozen=True)
class Grid:
    """Uniform n x n node grid (helmdd discretization.py:36-84)."""

    n: int
    bc: str

    def __post_init__(self):
        if self.n < 3:
            raise ValueError(f"need n >= 3 grid nodes per dimension, got {self.n}")
        if self.bc not in ("dirichlet", "sommerfeld"):
            raise ValueError(f"unknown boundary condition {self.bc!r}")

    @property
    def h(self) -> float:
        return 1.0 / (self.n - 1)

    @property
    def unknown_lo(self) -> int:
        return 1 if self.bc == "dirichlet" else 0

    @property
    def unknowns_per_dim(self) -> int:
        return self.n - 2 if self.bc == "dirichlet" else self.n

    @property
    def num_nodes(self) -> int:
        return self.n * self.n

    @property
    def num_unknowns(self) -> int:
        return self.unknowns_per_dim**2

    def unknown_index(self, ix, iy):
        lo = self.unknown_lo
        return (np.asarray(iy) - lo) * self.unknowns_per_dim + (np.asarray(ix) - lo)


@dataclass(frozen=True)
class RegimeReport:
    """Mesh-resolution products for (k, h, H) (helmdd discretization.py:97-121)."""

    kappa_h: float
    kappa_H: float
    pollution_metric: float

    _EPS = 1e-12

    @property
    def kappa_h_ok(self) -> bool:
        return self.kappa_h <= 0.25 + self._EPS

    @property
    def kappa_H_ok(self) -> bool:
        return self.kappa_H <= 1.0 + self._EPS

    @property
    def pollution_ok(self) -> bool:
        return self.pollution_metric <= 1.0 + self._EPS


def regime(k: float, h: float, H: float) -> RegimeReport:
    """helmdd discretization.py:124-127."""
    if k <= 0 or h <= 0 or H <= 0:
        raise ValueError("k, h, H must all be positive")
    return RegimeReport(kappa_h=k * h, kappa_H=k * H, pollution_metric=k**3 * h**2)


def pencil_1d(grid: Grid, k: float):
    """Dense 1-D pieces (T, w): A = T(x)W + W(x)T - k^2 W(x)W  (W = I for MP-1).

    T is the (-1,2,-1)/h^2 operator on the unknowns; Sommerfeld end rows are
    1/h^2 - ik/h with neighbour -1/h^2 and end weights 1/2
    (helmdd discretization.py:130-154, 171-188).
    """
    m, h = grid.unknowns_per_dim, grid.h
    dt = complex if grid.bc == "sommerfeld" else float
    T = np.zeros((m, m), dtype=dt)
    i = np.arange(m)
    T[i, i] = 2.0 / h**2
    T[i[:-1], i[:-1] + 1] = -1.0 / h**2
    T[i[1:], i[1:] - 1] = -1.0 / h**2
    w = np.ones(m)
    if grid.bc == "sommerfeld":
        T[0, 0] = T[-1, -1] = 1.0 / h**2 - 1j * k / h
        w[0] = w[-1] = 0.5
    return T, w


@dataclass(frozen=True)
class Partition:
    grid: Grid
    p: int

    @property
    def cells_per_subdomain(self) -> int:
        return (self.grid.n - 1) // self.p


def partition(grid: Grid, subdomains_per_dim: int) -> Partition:
    """p x p box partition (helmdd decomposition.py:89-103)."""
    p = subdomains_per_dim
    if p < 1:
        raise ValueError(f"need at least one subdomain per dimension, got {p}")
    if (grid.n - 1) % p != 0:
        raise ValueError(f"{p} subdomains per dimension do not divide {grid.n - 1} cells")
    return Partition(grid, p)


@dataclass(frozen=True)
class Decomposition:
    """Overlapping boxes with partition-of-unity weights (helmdd decomposition.py:46-63, 111-134)."""

    grid: Grid
    p: int
    overlap_layers: int

    @property
    def num_subdomains(self) -> int:
        return self.p * self.p

    @property
    def cells_per_subdomain(self) -> int:
        return (self.grid.n - 1) // self.p

    def interval(self, a: int):
        """Unknown-index interval [start, start+len) of 1-D box a (decomposition.py:66-79)."""
        g, c, m = self.grid, self.cells_per_subdomain, self.overlap_layers
        if m == 0:
            lo, hi = a * c + (1 if a > 0 else 0), (a + 1) * c
        else:
            lo, hi = a * c - (m - 1), (a + 1) * c + (m - 1)
        lo, hi = max(lo, g.unknown_lo), min(hi, g.unknown_lo + g.unknowns_per_dim - 1)
        return lo - g.unknown_lo, hi - lo + 1

    @cached_property
    def boxes(self):
        return [self.interval(a) for a in range(self.p)]

    @cached_property
    def multiplicity_1d(self) -> np.ndarray:
        m = np.zeros(self.grid.unknowns_per_dim, dtype=np.int64)
        for s, L in self.boxes:
            m[s : s + L] += 1
        return m

    @cached_property
    def multiplicity(self) -> np.ndarray:
        m = self.multiplicity_1d.astype(float)
        return np.outer(m, m).ravel()

    @cached_property
    def index_sets(self):
        nu = self.grid.unknowns_per_dim
        out = []
        for ys, yl in self.boxes:
            for xs, xl in self.boxes:
                iy, ix = np.mgrid[ys : ys + yl, xs : xs + xl]
                out.append((iy * nu + ix).ravel())
        return out

    @cached_property
    def weights(self):
        mult = self.multiplicity
        return [1.0 / mult[s] for s in self.index_sets]


def extend(part: Partition, overlap_layers: int, enforce_max_multiplicity: bool = False) -> Decomposition:
    """Grow the boxes by m layers (helmdd decomposition.py:111-134)."""
    if overlap_layers < 0:
        raise ValueError(f"overlap layer count must be nonnegative, got {overlap_layers}")
    dec = Decomposition(part.grid, part.p, overlap_layers)
    if enforce_max_multiplicity and dec.multiplicity_1d.max() ** 2 > 4:
        raise ValueError("overlap puts a node in more than 4 subdomains")
    return dec


def max_overlap_layers(part: Partition) -> int:
    return part.cells_per_subdomain // 2


def extend_max(part: Partition) -> Decomposition:
    return extend(part, max_overlap_layers(part), enforce_max_multiplicity=True)


def _check_ratio(grid: Grid, ratio: int, powers_of_two: bool):
    """coarse.py:77-81."""
    if ratio < 1 or (grid.n - 1) % ratio != 0:
        raise ValueError(f"coarsening ratio {ratio} does not divide {grid.n - 1} cells")
    if powers_of_two and ratio & (ratio - 1):
        raise ValueError(f"Bezier coarse space needs a power-of-two ratio, got {ratio}")


def bezier_1d(grid: Grid, ratio: int = 2) -> np.ndarray:
    """Dense 1-D Bezier restriction P (m0 x nu): the one-level (1,4,6,4,1)/8 stride-2 stencil
    composed through the intermediate grids, taps outside each level's unknown set dropped
    (helmdd coarse.py:102-133; Dirichlet levels keep their interior nodes only)."""
    _check_ratio(grid, ratio, powers_of_two=True)
    taps = np.array([1.0, 4.0, 6.0, 4.0, 1.0]) / 8.0
    dirichlet = grid.bc == "dirichlet"
    op = None
    nf = grid.n
    for _ in range(int(round(np.log2(ratio)))):
        M = (nf + 1) // 2
        if dirichlet:  # unknowns: interior nodes 1..nf-2 -> coarse interior 1..M-2
            S = np.zeros((M - 2, nf - 2))
            for I in range(1, M - 1):
                for d in range(-2, 3):
                    i = 2 * I + d
                    if 1 <= i <= nf - 2:
                        S[I - 1, i - 1] = taps[d + 2]
        else:
            S = np.zeros((M, nf))
            for I in range(M):
                for d in range(-2, 3):
                    i = 2 * I + d
                    if 0 <= i < nf:
                        S[I, i] = taps[d + 2]
        op = S if op is None else S @ op
        nf = M
    return op


def hat_1d(grid: Grid, ratio: int) -> np.ndarray:
    """Dense 1-D hat-function sampling matrix (helmdd coarse.py:84-99): weights 1 - |d|/r
    around every r-th node; Dirichlet drops the boundary coarse nodes and fine columns."""
    _check_ratio(grid, ratio, powers_of_two=False)
    n, r = grid.n, ratio
    M = (n - 1) // r + 1
    P = np.zeros((M, n))
    for J in range(M):
        for d in range(-r + 1, r):
            i = r * J + d
            if 0 <= i < n:
                P[J, i] = 1.0 - abs(d) / r
    if grid.bc == "dirichlet":
        P = P[1:-1, 1:-1]
    return np.ascontiguousarray(P)


@dataclass(frozen=True)
class CoarseSpace:
    """Coarse space descriptor (helmdd coarse.py:42-74): kind FOCS / HOCS at H = ratio*h.
    ``fdm`` holds the coarse-solver setup once :func:`galerkin` has run."""

    kind: str
    grid: Grid
    ratio: int
    fdm: object = field(default=None, compare=False, repr=False)

    @property
    def coarse_nodes_per_dim(self) -> int:
        return (self.grid.n - 1) // self.ratio + 1

    @property
    def coarse_unknowns_per_dim(self) -> int:
        m = self.coarse_nodes_per_dim
        return m - 2 if self.grid.bc == "dirichlet" else m

    @property
    def coarse_size(self) -> int:
        """All-node count of the coarse grid (coarse.py:61-63)."""
        return self.coarse_nodes_per_dim**2

    @property
    def num_coarse_unknowns(self) -> int:
        return self.coarse_unknowns_per_dim**2

    def restriction_1d(self) -> np.ndarray:
        """The dense 1-D P with R0 = P (x) P (coarse.py:136-139)."""
        return bezier_1d(self.grid, self.ratio) if self.kind == "HOCS" else hat_1d(self.grid, self.ratio)


def build_hocs(grid: Grid, ratio: int) -> CoarseSpace:
    """Bezier coarse space with H = ratio*h, ratio in 2, 4, 8, 16 (helmdd coarse.py:148-151)."""
    _check_ratio(grid, ratio, powers_of_two=True)
    return CoarseSpace("HOCS", grid, ratio)


def build_focs(grid: Grid, ratio: int) -> CoarseSpace:
    """Linear (bilinear hat) coarse space with H = ratio*h (helmdd coarse.py:142-145)."""
    _check_ratio(grid, ratio, powers_of_two=False)
    return CoarseSpace("FOCS", grid, ratio)
