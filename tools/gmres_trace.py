"""Per-iteration host trace of the device GMRES (HELM_GMRES_TRACE=1), run several times back to back."""
import os
import subprocess
import sys
import threading
import time
os.environ["HELM_GMRES_TRACE"] = "1"
sys.path.insert(0, ".")
import paper_2408_03571_b200 as hb

n, k, p, iters, runs = 2049, 300.0, 64, int(sys.argv[1]), int(sys.argv[2])
grid = hb.Grid(n, "sommerfeld")
prob = hb.assemble(grid, k, "MP2")
M = hb.SchwarzPreconditioner("SHS2", prob.A, hb.extend(hb.partition(grid, p), 2), hb.galerkin(hb.build_hocs(grid, 2), prob.A))
samples = []
stop = False


def smi():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader"],
                             capture_output=True, text=True).stdout.strip()
        samples.append((time.time(), out))
        time.sleep(0.05)


th = threading.Thread(target=smi, daemon=True)
th.start()
for r in range(runs):
    t = time.time()
    rep = hb.gmres(prob.A, M, prob.f, hb.GmresConfig(rtol=1e-30, max_iter=iters))
    print("run", r, rep.iterations, rep.wall_seconds, "start", t, file=sys.stderr, flush=True)
stop = True
th.join()
for s in samples:
    print("smi %.3f %s" % s, file=sys.stderr)
