"""Shared helpers for the parity tests: golden fixtures and seeded inputs."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def golden_names(store_vectors=True):
    out = []
    for f in sorted(os.listdir(GOLDEN)):
        if f.endswith(".npz") and not f.endswith("_ops.npz"):  # *_ops: sampled large-config goldens
            g = np.load(os.path.join(GOLDEN, f))
            if ("M_shs2" in g.files) == store_vectors:
                out.append(f[:-4])
    return out


def operator_input(N, complex_):
    """Seed-1 operator input: real block drawn first, then the imaginary block."""
    r = np.random.default_rng(1)
    x = r.standard_normal(N)
    return x + 1j * r.standard_normal(N) if complex_ else x


def random_rhs(N):
    r = np.random.default_rng(0)
    return r.standard_normal(N) + 1j * r.standard_normal(N)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def reference_count(name, g):
    """The unmodified reference's raw GMRES count (gmres.py:65-177, its golden run)."""
    return int(g["gmres_iterations"])


def _spread(name):
    path = os.path.join(GOLDEN, name + "_spread.json")
    if not os.path.exists(path):
        return []
    import json

    with open(path) as f:
        return json.load(f)["runs"]


def raw_reference_counts(name, g):
    """Counts of the UNMODIFIED reference under the choices its specification leaves open
    (SuperLU column ordering, subdomain order; tests/golden/make_spread.py), with its golden run."""
    return sorted({int(g["gmres_iterations"])} | {r["iterations"] for r in _spread(name)
                                                  if r.get("coarse", "superlu") == "superlu"})


def accurate_reference_counts(name):
    """Counts of the reference's own GMRES loop and preconditioner with its inner solves made
    ACCURATE (SuperLU + iterative refinement, the exact transform coarse solve, fast-diagonalisation
    local solves: make_spread.py / make_refined.py), i.e. what the algorithm gives once the rounding
    of the reference's SuperLU solves (~1e-13 relative at cfg3 / cfg4a) is taken out."""
    import json

    out = {r["iterations"] for r in _spread(name) if r.get("coarse", "superlu") != "superlu"}
    for tag in ("_exact", "_refined"):
        path = os.path.join(GOLDEN, name + tag + ".json")
        if os.path.exists(path):
            with open(path) as f:
                out.add(int(json.load(f)["iterations"]))
    return sorted(out)


def reference_solution_spread(name, g):
    """Largest relative difference, on the golden's sampled iterate, between the reference's own
    solutions under the SPEC-allowed variations (same count bar; make_spread.py stores every
    97th sample of the golden's sample)."""
    ref = g["gmres_x_sample"][::97]
    worst = 0.0
    for r in _spread(name):
        if r.get("coarse", "superlu") != "superlu":
            continue
        x = np.array([a + 1j * b for a, b in r["x_sample"]])
        worst = max(worst, float(np.linalg.norm(x - ref) / np.linalg.norm(ref)))
    return worst


def count_matches(it, raw):
    """Iteration-count bar (north star: +-1 of the reference)."""
    return abs(it - raw) <= 1
