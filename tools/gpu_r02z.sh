#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu -s tests/test_gpu_ozaki.py tests/test_gpu_parity.py -k "ring_depth or four_rhs" 2>&1 | tail -15
