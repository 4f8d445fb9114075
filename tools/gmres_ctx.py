"""Does prior batch-32 / pinned-host work slow the fixed-length GMRES down? (development probe)"""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

grid = hb.Grid(2049, "sommerfeld"); prob = hb.assemble(grid, 300.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 64), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A), max_batch=32)
N = prob.A.N
r0 = np.random.default_rng(0)
b = r0.standard_normal(N) + 1j * r0.standard_normal(N)
cfg = hb.GmresConfig(rtol=1e-300, max_iter=50)
def fixed(tag):
    hb.gmres(prob.A, M, b, cfg)
    rep = hb.gmres(prob.A, M, b, cfg)
    print(f"{tag}: {1e3 * rep.wall_seconds / rep.iterations:.4f} ms/it", flush=True)
fixed("fresh")
X = torch.randn(32, N, dtype=torch.complex128, device="cuda")
Y = torch.empty_like(X)
for _ in range(20):
    M(X, out=Y)
torch.cuda.synchronize()
fixed("after 20 batch-32 applies")
Xh = torch.empty((32, N), dtype=torch.complex128, pin_memory=True)
Yh = torch.empty_like(Xh).pin_memory()
for _ in range(3):
    M.apply(Xh, out=Yh)
torch.cuda.synchronize()
fixed("after pinned e2e applies")
del Xh, Yh
fixed("after freeing the pinned buffers")
del X, Y
torch.cuda.empty_cache()
fixed("after freeing the device batch")
