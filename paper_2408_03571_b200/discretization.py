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
    def num_unknowns(self) -> int:
        return self.unknowns_per_dim**2

    def unknown_index(self, ix, iy):
        lo = self.unknown_lo
        return (np.asarray(iy) - lo) * self.unknowns_per_dim + (np.asarray(ix) - lo)


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


def bezier_1d(grid: Grid, ratio: int = 2) -> np.ndarray:
    """Dense 1-D Bezier restriction P (m0 x nu): (1,4,6,4,1)/8 at stride 2, taps
    outside the unknown set dropped (helmdd coarse.py:102-133).  Ratio 2 only."""
    if ratio != 2:
        raise NotImplementedError("only the HOCS ratio H = 2h is implemented on the GPU path")
    nu = grid.unknowns_per_dim
    off = grid.unknown_lo
    m0 = (grid.n - 3) // 2 if grid.bc == "dirichlet" else (grid.n + 1) // 2
    taps = np.array([1.0, 4.0, 6.0, 4.0, 1.0]) / 8.0
    P = np.zeros((m0, nu))
    for d in range(-2, 3):
        U = np.arange(m0)
        u = 2 * U + off + d
        ok = (u >= 0) & (u < nu)
        P[U[ok], u[ok]] = taps[d + 2]
    return P


@dataclass(frozen=True)
class CoarseSpace:
    """HOCS coarse space descriptor (helmdd coarse.py:42-74); ``fdm`` holds the
    partial-FDM setup once :func:`galerkin` has run."""

    kind: str
    grid: Grid
    ratio: int
    fdm: object = field(default=None, compare=False, repr=False)

    @property
    def coarse_unknowns_per_dim(self) -> int:
        g = self.grid
        return (g.n - 3) // 2 if g.bc == "dirichlet" else (g.n + 1) // 2

    @property
    def num_coarse_unknowns(self) -> int:
        return self.coarse_unknowns_per_dim**2


def build_hocs(grid: Grid, ratio: int) -> CoarseSpace:
    """Bezier coarse space with H = ratio*h (helmdd coarse.py:148-151); ratio 2 only."""
    if ratio < 1 or (grid.n - 1) % ratio != 0:
        raise ValueError(f"coarsening ratio {ratio} does not divide {grid.n - 1} cells")
    if ratio & (ratio - 1):
        raise ValueError(f"Bezier coarse space needs a power-of-two ratio, got {ratio}")
    if ratio != 2:
        raise NotImplementedError("only the HOCS ratio H = 2h is implemented on the GPU path")
    return CoarseSpace("HOCS", grid, ratio)
