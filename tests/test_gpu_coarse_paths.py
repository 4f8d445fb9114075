"""Coarse-solve kernel paths selected by environment switches (read once per process, so each
variant runs in its own interpreter): the TMA-staged band kernel against the cp.async kernel
(bitwise), the strip-first pass order against the round-1 order (rounding level), both against
A0 y = c.  Reference operation: linalg.solve(cs.a0_factorization, c), coarse.py:174."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2408_03571_b200 as hb
n, k, p, B, out = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
grid = hb.Grid(n, "sommerfeld")
prob = hb.assemble(grid, k, "MP2")
dec = hb.extend(hb.partition(grid, p), 2)
cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, max_batch=B)
rng = np.random.default_rng(5)
C = rng.standard_normal((B, M.N0)) + 1j * rng.standard_normal((B, M.N0))
X = rng.standard_normal((B, M.N)) + 1j * rng.standard_normal((B, M.N))
Y = M.coarse_solve(torch.from_numpy(C).cuda()).cpu().numpy()
Z = M(torch.from_numpy(X).cuda()).cpu().numpy()
np.savez(out, C=C, Y=Y, Z=Z)
""" % ROOT


def run(tmp_path, tag, env, n, k, p, B):
    out = str(tmp_path / f"{tag}.npz")
    r = subprocess.run([sys.executable, "-c", CHILD, str(n), str(k), str(p), str(B), out],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n,k,p,B", [(65, 10.0, 4, 5), (129, 30.0, 8, 17), (257, 50.0, 8, 13), (513, 100.0, 16, 8)])
def test_tma_band_kernel_is_bitwise_the_cp_async_kernel(tmp_path, n, k, p, B):
    """band_tma.cu stages the same chunks with bulk / tensor copies and runs the same recurrence
    in the same order: the results must be identical, including a batch that is not a multiple of
    the 8 right-hand sides a CTA owns (zero-filled by the TMA unit)."""
    a = run(tmp_path, "tma", {"HELM_BAND_TMA": "1"}, n, k, p, B)
    b = run(tmp_path, "cpasync", {"HELM_BAND_TMA": "0"}, n, k, p, B)
    assert np.array_equal(a["Y"], b["Y"]) and np.array_equal(a["Z"], b["Z"])


def test_strip_first_order_matches_full_passes(tmp_path):
    """Strip-first order (two strip-value passes + one full pass) against the round-1 order
    (three full passes + strip sweeps): the same linear algebra associated differently."""
    import scipy.sparse as sp

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import helmdd_oracle as O  # checker only: A0 = R0 A R0^T

    n, k, p, B = 257, 50.0, 8, 8
    a = run(tmp_path, "first", {"HELM_STRIP_FIRST": "1"}, n, k, p, B)
    b = run(tmp_path, "full", {"HELM_STRIP_FIRST": "0"}, n, k, p, B)
    assert rel(a["Y"], b["Y"]) <= 1e-13 and rel(a["Z"], b["Z"]) <= 1e-13
    og = O.OGrid(n, "sommerfeld")
    oprob = O.assemble(og, k, "MP2")
    P1 = O.bezier_1d(og, 2)
    r0 = sp.kron(P1, P1, format="csr").astype(complex)
    a0 = (r0 @ oprob.A @ r0.T).tocsr()
    for i in (0, B - 1):
        assert np.linalg.norm(a0 @ a["Y"][i] - a["C"][i]) / np.linalg.norm(a["C"][i]) <= 1e-12
