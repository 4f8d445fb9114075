"""GMRES wall time vs iteration cap on the config-5 operator with the seed-0 random RHS."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

grid = hb.Grid(2049, "sommerfeld")
prob = hb.assemble(grid, 300.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 64), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A))
r = np.random.default_rng(0)
b = r.standard_normal(prob.A.N) + 1j * r.standard_normal(prob.A.N)
import torch
bd = torch.from_numpy(b).cuda()
hb.gmres(prob.A, M, bd, hb.GmresConfig(rtol=1e-30, max_iter=60))
prev = 0.0
for cap in (1, 2, 5, 10, 20, 30, 40, 50):
    rep = hb.gmres(prob.A, M, bd, hb.GmresConfig(rtol=1e-30, max_iter=cap))
    rep2 = hb.gmres(prob.A, M, b, hb.GmresConfig(rtol=1e-30, max_iter=cap))
    print("cap %3d: device-b %.2f ms (%.3f ms/it)   host-b %.2f ms" % (cap, rep.wall_seconds * 1e3, rep.wall_seconds * 1e3 / cap, rep2.wall_seconds * 1e3), flush=True)
