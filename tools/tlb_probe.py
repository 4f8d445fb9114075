"""Does a large sweep between batch-1 M^-1 applies slow the apply down? (development probe)"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

grid = hb.Grid(2049, "sommerfeld")
prob = hb.assemble(grid, 300.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 64), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A))
lib, pl = M.plan.lib, M.plan
st = torch.cuda.current_stream()
N = M.N
x = torch.randn(N, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
c = torch.randn(M.N0, dtype=torch.complex128, device="cuda")
c2 = torch.empty_like(c)


def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


Mf = lambda: lib.helm_apply_M(pl.handle, pl.ws, x.data_ptr(), y.data_ptr(), 1, st.cuda_stream)
Cf = lambda: lib.helm_coarse_solve(pl.handle, pl.ws, c.data_ptr(), c2.data_ptr(), 1, st.cuda_stream)
print("M alone %.3f  coarse alone %.3f" % (ev(Mf), ev(Cf)))
for gb in (0.5, 1, 1.5, 2, 2.5, 3, 4, 6):
    big = torch.empty(int(gb * 2**30) // 8, dtype=torch.float64, device="cuda")
    sw = lambda: big.fill_(1.0)
    ts = ev(sw)
    tm = ev(lambda: (sw(), Mf()))
    tc = ev(lambda: (sw(), Cf()))
    print("sweep %.1f GB: sweep %.3f  sweep+M %.3f -> M %.3f ; coarse %.3f" % (gb, ts, tm, tm - ts, tc - ts))
    del big
