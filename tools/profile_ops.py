"""Per-operator device timings at a BASELINE config (CUDA events; development tool)."""

import argparse
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb  # noqa: E402


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2049)
    ap.add_argument("--k", type=float, default=300.0)
    ap.add_argument("--p", type=int, default=64)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--gmres", type=int, default=30)
    ap.add_argument("--only", default="", help="comma-separated op names to time (default: all)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--batches", default="1,32")
    ap.add_argument("--setup", default="native", help="native | host (host: no cuSOLVER kernels, quick under ncu)")
    a = ap.parse_args()
    t = time.time()
    grid = hb.Grid(a.n, "sommerfeld")
    prob = hb.assemble(grid, a.k, "MP2")
    dec = hb.extend(hb.partition(grid, a.p), 2)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, max_batch=a.batch, setup=a.setup)
    print(f"setup {time.time() - t:.1f}s", flush=True)
    N, N0 = M.N, M.N0
    p, lib = M.plan, M.plan.lib
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    for B in [int(v) for v in a.batches.split(",")]:
        X = torch.randn(B, N, dtype=torch.complex128, device="cuda")
        Y = torch.empty_like(X)
        C = torch.randn(B, N0, dtype=torch.complex128, device="cuda")
        C2 = torch.empty_like(C)
        ops = {
            "A x": lambda: lib.helm_apply_A(p.handle, X.data_ptr(), Y.data_ptr(), B, st()),
            "R0 x": lambda: lib.helm_restrict(p.handle, X.data_ptr(), C.data_ptr(), B, st()),
            "R0^T c": lambda: lib.helm_prolong(p.handle, C.data_ptr(), Y.data_ptr(), B, st()),
            "coarse solve": lambda: lib.helm_coarse_solve(p.handle, p.ws, C.data_ptr(), C2.data_ptr(), B, st()),
            "local sum": lambda: lib.helm_local_sum(p.handle, p.ws, X.data_ptr(), None, Y.data_ptr(), 1, B, st()),
            "M^-1": lambda: lib.helm_apply_M(p.handle, p.ws, X.data_ptr(), Y.data_ptr(), B, st()),
        }
        for name, fn in ops.items():
            if a.only and name not in a.only.split(","):
                continue
            ms = timeit(fn, reps=a.reps, warm=min(2, a.reps))
            print(f"B={B:3d} {name:14s} {ms:9.3f} ms  ({ms / B:8.3f} ms/vec)", flush=True)
    if a.gmres:
        rep = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-6, max_iter=a.gmres))
        print(f"GMRES {rep.iterations} it in {rep.wall_seconds:.3f}s -> {rep.iterations / rep.wall_seconds:.1f} it/s, "
              f"est {rep.residual_history[-1]:.3e}")


if __name__ == "__main__":
    main()
