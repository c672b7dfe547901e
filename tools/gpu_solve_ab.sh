#!/bin/bash
# solve parity tests, then the C4 4-RHS sweep with scalar (0) and tensor-core small-front kernels (1)
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_verify.py tests/test_gpu_factor_structure.py 2>&1 | tail -3
for v in 0 1; do echo "RBA_BWD_MMA=$v"; RBA_BWD_MMA=$v timeout 300 python tools/solve_check.py 3 2>&1 | tail -4; done
