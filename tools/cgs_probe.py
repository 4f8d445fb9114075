import sys, torch
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb
grid = hb.Grid(129, "sommerfeld")
prob = hb.assemble(grid, 20.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 8), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A))
lib, pl = M.plan.lib, M.plan
N = M.N
st = torch.cuda.current_stream()
for j in (100, 200, 215, 216, 217, 250, 300, 383, 384, 385, 500, 700, 999):
    V = torch.randn(j + 2, N, dtype=torch.complex128, device="cuda")
    h = torch.empty(j + 2, dtype=torch.complex128, device="cuda")
    s = lib.helm_cgs2(pl.handle, pl.ws, V.data_ptr(), j, h.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    print(j, s, lib.helm_last_error().decode() if s else "", flush=True)
