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
        if f.endswith(".npz"):
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
