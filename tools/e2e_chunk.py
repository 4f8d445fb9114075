"""e2e (pinned host batch -> host batch) M^-1 applies/s at config 5 vs the pipeline chunk size
(development tool)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

grid = hb.Grid(2049, "sommerfeld"); prob = hb.assemble(grid, 300.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 64), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A), max_batch=32)
B, N = 32, prob.A.N
Xh = torch.empty((B, N), dtype=torch.complex128, pin_memory=True)
Xh.copy_(torch.randn(B, N, dtype=torch.complex128))
Yh = torch.empty_like(Xh).pin_memory()
for c in [int(v) for v in sys.argv[1:]] or [2, 4, 8, 16]:
    hb.SchwarzPreconditioner.PIPE_CHUNK = c
    M._pipe = None
    M.apply(Xh, out=Yh); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        M.apply(Xh, out=Yh)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"chunk {c}: {B / dt:.1f} applies/s ({1e3 * dt:.1f} ms per batch of {B})", flush=True)
