mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/pytest_multi.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_multi.log
cat > /tmp/mb.py <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb
grid = hb.Grid(2049, "sommerfeld"); prob = hb.assemble(grid, 300.0, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, 64), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A), max_batch=8)
r = np.random.default_rng(0)
for nr in (1, 2, 4, 8):
    B = r.standard_normal((nr, prob.A.N)) + 1j * r.standard_normal((nr, prob.A.N))
    cfg = hb.GmresConfig(rtol=1e-300, max_iter=50)
    hb.gmres_multi(prob.A, M, B, cfg)
    reps = hb.gmres_multi(prob.A, M, B, cfg)
    w = reps[0].wall_seconds
    print(f"nrhs {nr}: {sum(q.iterations for q in reps)} RHS-iterations in {w:.3f} s -> {sum(q.iterations for q in reps)/w:.1f} it/s, {1e3*w/50:.3f} ms per batched iteration", flush=True)
PY
timeout 900 python /tmp/mb.py
