"""A/B of the fast-sine box kernel (local_dst.cu) against the DMMA box kernel (HELM_DST=0):
local sum and M^-1 agreement and timings on MP-1 / MP-2 configs (development tool, GPU)."""

import os
import sys

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


def build(n, k, p, bc, B, dst):
    os.environ["HELM_DST"] = "1" if dst else "0"
    os.environ["HELM_EDGE"] = "1" if dst else "0"
    grid = hb.Grid(n, bc)
    prob = hb.assemble(grid, k, "MP2" if bc == "sommerfeld" else "MP1")
    dec = hb.extend(hb.partition(grid, p), 2)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    return hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, max_batch=B)


def main():
    cfgs = [(65, 20.0, 4, "dirichlet", 4), (65, 10.0, 4, "sommerfeld", 4), (257, 50.0, 8, "sommerfeld", 5),
            (513, 100.0, 16, "dirichlet", 3), (2049, 300.0, 64, "sommerfeld", 32)]
    if len(sys.argv) > 1:
        cfgs = [c for c in cfgs if str(c[0]) in sys.argv[1].split(",")]
    for n, k, p, bc, B in cfgs:
        res = {}
        for dst in (False, True):
            M = build(n, k, p, bc, B, dst)
            pl, lib = M.plan, M.plan.lib
            st = torch.cuda.current_stream().cuda_stream
            dt = torch.complex128 if bc == "sommerfeld" else torch.float64
            g = torch.Generator(device="cuda").manual_seed(7)
            X = torch.randn(B, M.N, dtype=dt, device="cuda", generator=g)
            Y = torch.empty_like(X)
            Z = torch.empty_like(X)
            ls = lambda: lib.helm_local_sum(pl.handle, pl.ws, X.data_ptr(), None, Y.data_ptr(), 1, B, st)  # noqa
            mi = lambda: lib.helm_apply_M(pl.handle, pl.ws, X.data_ptr(), Z.data_ptr(), B, st)  # noqa
            ls()
            mi()
            torch.cuda.synchronize()
            tl = timeit(ls, reps=5 if n > 1000 else 20)
            tm = timeit(mi, reps=5 if n > 1000 else 20)
            res[dst] = (Y.clone(), Z.clone(), tl, tm)
            del M
        (y0, z0, tl0, tm0), (y1, z1, tl1, tm1) = res[False], res[True]
        el = (torch.linalg.norm(y1 - y0) / torch.linalg.norm(y0)).item()
        em = (torch.linalg.norm(z1 - z0) / torch.linalg.norm(z0)).item()
        print(f"n={n} {bc} p={p} B={B}: local sum diff {el:.2e}, M^-1 diff {em:.2e}; "
              f"local sum {tl0:.3f} -> {tl1:.3f} ms, M^-1 {tm0:.3f} -> {tm1:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
