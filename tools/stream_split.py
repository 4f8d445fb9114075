"""Experiment: SHS2 M^-1 on a batch of 32 as two half-batches on two streams (two workspaces)."""
import ctypes
import sys
import torch
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

grid = hb.Grid(2049, "sommerfeld")
prob = hb.assemble(grid, 300.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 64), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A), max_batch=32)
lib, pl = M.plan.lib, M.plan
N = M.N
wss = []
for _ in range(4):
    w = ctypes.c_void_p()
    assert lib.helm_workspace_create(pl.handle, 16, ctypes.byref(w)) == 0
    wss.append(w)
X = torch.randn(32, N, dtype=torch.complex128, device="cuda")
Y = torch.empty_like(X)
s0 = torch.cuda.current_stream()
streams = [torch.cuda.Stream() for _ in range(4)]


def one():
    lib.helm_apply_M(pl.handle, pl.ws, X.data_ptr(), Y.data_ptr(), 32, s0.cuda_stream)


def split(k):
    B = 32 // k
    ev = torch.cuda.Event()
    ev.record(s0)
    for i in range(k):
        streams[i].wait_event(ev)
        off = i * B * N * 16
        lib.helm_apply_M(pl.handle, wss[i], X.data_ptr() + off, Y.data_ptr() + off, B, streams[i].cuda_stream)
    for i in range(k):
        e = torch.cuda.Event()
        e.record(streams[i])
        s0.wait_event(e)


def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s0)
    for _ in range(reps):
        fn()
    b.record(s0); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


print("1 x 32: %.3f ms" % t(one))
print("2 x 16: %.3f ms" % t(lambda: split(2)))
print("4 x 8 : %.3f ms" % t(lambda: split(4)))
