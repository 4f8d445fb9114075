import sys
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb
n, k, p, iters = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
grid = hb.Grid(n, "sommerfeld")
prob = hb.assemble(grid, k, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, p), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A))
rep = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-30, max_iter=iters))
print(rep.iterations, rep.wall_seconds)
