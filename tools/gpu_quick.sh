# quick check: GPU parity tests (no large GMRES runs) + per-operator timings at config 5
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not large" > gpurun_out/pytest_quick.log 2>&1; echo pytest=$?
timeout 600 python tools/profile_ops.py --gmres 0 --reps 5 --only "${1:-local sum,coarse solve,M^-1}" > gpurun_out/ops.log 2>&1; echo ops=$?
