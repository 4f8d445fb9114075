"""Per-iteration cost of the device GMRES at a BASELINE config (development tool): times a fixed
number of iterations and the pieces of one iteration (M^-1, A x, CGS2 at basis size j) with CUDA events."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb
from paper_2408_03571_b200 import _lib

n, k, p = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 50
grid = hb.Grid(n, "sommerfeld")
prob = hb.assemble(grid, k, "MP2")
dec = hb.extend(hb.partition(grid, p), 2)
M = hb.SchwarzPreconditioner("SHS2", prob.A, dec, hb.galerkin(hb.build_hocs(grid, 2), prob.A))
N = M.N
lib, pl = M.plan.lib, M.plan
st = torch.cuda.current_stream()


def ev_time(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


x = torch.randn(N, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
print("M^-1 (B=1)  %.3f ms" % ev_time(lambda: lib.helm_apply_M(pl.handle, pl.ws, x.data_ptr(), y.data_ptr(), 1, st.cuda_stream)))
print("A x (B=1)   %.3f ms" % ev_time(lambda: lib.helm_apply_A(pl.handle, x.data_ptr(), y.data_ptr(), 1, st.cuda_stream)))
for j in (0, 9, 24, 49):
    V = torch.randn(j + 2, N, dtype=torch.complex128, device="cuda")
    h = torch.empty(j + 2, dtype=torch.complex128, device="cuda")
    print("CGS2 j=%3d  %.3f ms" % (j, ev_time(lambda: lib.helm_cgs2(pl.handle, pl.ws, V.data_ptr(), j, h.data_ptr(), st.cuda_stream))))
    del V
for b in (prob.f,):
    rep = hb.gmres(prob.A, M, b, hb.GmresConfig(rtol=1e-30, max_iter=iters))
    rep = hb.gmres(prob.A, M, b, hb.GmresConfig(rtol=1e-30, max_iter=iters))
    print("GMRES %d iterations: %.3f s -> %.1f it/s (%.3f ms/it)" % (rep.iterations, rep.wall_seconds,
          rep.iterations / rep.wall_seconds, 1e3 * rep.wall_seconds / rep.iterations))
