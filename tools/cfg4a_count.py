"""Device GMRES iteration count for BASELINE config 4(a) (n=1025, k=200, point source) under the
coarse-solve accuracy options given on the command line: refine_steps strip_refine (development tool;
the env switches HELM_BAND_SEG_MAX / HELM_BAND_NOPIV select other kernel paths)."""
import sys
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

ir = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sr = int(sys.argv[2]) if len(sys.argv) > 2 else 1
grid = hb.Grid(1025, "sommerfeld")
prob = hb.assemble(grid, 200.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 32), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A),
                             refine_steps=ir, strip_refine=sr)
rep = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-6, max_iter=1000))
print("cfg4a refine", ir, "strip", sr, "iterations", rep.iterations, rep.converged, rep.final_residual)
