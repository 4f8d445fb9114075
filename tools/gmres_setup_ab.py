"""GMRES wall time at config 5 with the host and the native setup (development probe, GPU)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb  # noqa: E402

n, k, p = 2049, 300.0, 64
grid = hb.Grid(n, "sommerfeld")
prob = hb.assemble(grid, k, "MP2")
dec = hb.extend(hb.partition(grid, p), 2)
cs = hb.galerkin(hb.build_hocs(grid, 2), prob.A)
for setup in sys.argv[1:] or ["host", "native"]:
    for mb in (1, 32):
        M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, cs, max_batch=mb, setup=setup)
        for rep_i in range(3):
            t = time.time()
            rep = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-6, max_iter=100))
            print(f"setup={setup} max_batch={mb} run {rep_i}: {rep.iterations} it, lib wall {rep.wall_seconds*1e3:.2f} ms, "
                  f"py wall {(time.time()-t)*1e3:.2f} ms", flush=True)
        X = torch.zeros(1, M.N, dtype=torch.complex128, device="cuda")
        X[0, 0] = 1
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            M(X)
        e1.record()
        torch.cuda.synchronize()
        print(f"   M^-1 batch 1: {e0.elapsed_time(e1)/10:.3f} ms", flush=True)
        del M
