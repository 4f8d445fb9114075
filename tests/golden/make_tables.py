"""Paper-table goldens from the UNMODIFIED reference harness (build container only).

Runs ``helmdd.harness.run_experiment`` on the built-in table sweeps (harness.py:272-314), restricted
the way the reference's acceptance suite restricts them (pkg/tests/test_acceptance.py:37-131), and
stores every cell's iteration count ("x" = not converged) in tests/golden/paper_tables.json.  The
device harness (paper_2408_03571_b200/harness.py, backend "b200") must reproduce them within +-1
(tests/test_gpu_coarse_spaces.py).

Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_tables.py
"""

from __future__ import annotations

import json
import os
import time
from dataclasses import replace

HERE = os.path.dirname(os.path.abspath(__file__))
KS = (20, 40, 60, 80, 100)

# (table, overrides) -- test_acceptance.py criteria 1-5
SWEEPS = [
    (1, dict(k_list=KS, n_list=tuple(4 * k + 1 for k in KS))),                      # MP-2, FOCS + HOCS, all kinds
    (2, dict(k_list=KS, n_list=tuple(4 * k + 1 for k in KS))),                      # MP-1, FOCS + HOCS, all kinds
    (3, dict(k_list=(10, 20), n_list=tuple(range(33, 162, 8)))),                     # MP-1 HOCS H=4h sweep
    (4, dict(k_list=(5, 30), n_list=(33, 49, 65, 81, 97, 113, 129, 257))),           # MP-1 HOCS H=16h
]


def main():
    from helmdd.harness import builtin_table, run_experiment

    out = []
    for table, ov in SWEEPS:
        cfg = replace(builtin_table(table), **ov)
        t0 = time.time()
        rows = run_experiment(cfg, warn=lambda m: None)
        out.append(dict(table=table, problem=cfg.problem, ratio=cfg.coarse_ratio, overlap=cfg.overlap,
                        rtol=cfg.gmres.rtol, max_iter=cfg.gmres.max_iter, side=cfg.gmres.side,
                        seconds=round(time.time() - t0, 1),
                        rows=[dict(k=r.k, n=r.n, iterations=r.iterations) for r in rows]))
        print(json.dumps(out[-1]), flush=True)
    with open(os.path.join(HERE, "paper_tables.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
