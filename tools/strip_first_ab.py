"""A/B of the coarse-solve pass order (HELM_STRIP_FIRST=0/1) at config 5: coarse-solve and M^-1 timings at
batch 32 / 8, agreement of the two orders and the A0 residual (development tool, GPU).
Run as: python tools/strip_first_ab.py  (spawns itself once per order)."""
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, ".")


def timeit(fn, reps=10, warm=3):
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


def child(tag):
    import paper_2408_03571_b200 as hb

    n, k, p = 2049, 300.0, 64
    grid = hb.Grid(n, "sommerfeld")
    prob = hb.assemble(grid, k, "MP2")
    dec = hb.extend(hb.partition(grid, p), 2)
    cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
    M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, max_batch=32)
    pl, lib = M.plan, M.plan.lib
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(11)
    for B in (32, 13, 8):
        C = torch.randn(B, M.N0, dtype=torch.complex128, device="cuda", generator=g)
        Y = torch.empty_like(C)
        X = torch.randn(B, M.N, dtype=torch.complex128, device="cuda", generator=g)
        Z = torch.empty_like(X)
        cs_ = lambda: lib.helm_coarse_solve(pl.handle, pl.ws, C.data_ptr(), Y.data_ptr(), B, st)  # noqa
        mi = lambda: lib.helm_apply_M(pl.handle, pl.ws, X.data_ptr(), Z.data_ptr(), B, st)  # noqa
        tc, tm = timeit(cs_), timeit(mi)
        print(f"[{tag}] batch {B}: coarse solve {tc:.3f} ms, M^-1 {tm:.3f} ms", flush=True)
        torch.save((Y[:2].cpu(), Z[:2].cpu()), f"/tmp/sf_{tag}_{B}.pt")
        other = f"/tmp/sf_{'old' if tag == 'new' else 'new'}_{B}.pt"
        if os.path.exists(other):
            Yo, Zo = torch.load(other)
            ey = (torch.linalg.norm(Y[:2].cpu() - Yo) / torch.linalg.norm(Yo)).item()
            ez = (torch.linalg.norm(Z[:2].cpu() - Zo) / torch.linalg.norm(Zo)).item()
            print(f"   new vs old: coarse solve {ey:.2e}, M^-1 {ez:.2e}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child(sys.argv[1])
    else:
        # default: pass order A/B; "tma": the TMA-staged band kernel against the cp.async one
        var = "HELM_BAND_TMA" if os.environ.get("AB") == "tma" else "HELM_STRIP_FIRST"
        for tag, v in (("old", "0"), ("new", "1")):
            subprocess.run([sys.executable, __file__, tag], env=dict(os.environ, **{var: v}), check=False, timeout=400)
