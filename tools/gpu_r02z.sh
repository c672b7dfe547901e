#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_verify.py 2>&1 | tail -4
for v in 0 1; do echo "BWD_MMA=$v"; RBA_BWD_MMA=$v timeout 300 python tools/solve_check.py 3 2>&1 | tail -4; done
