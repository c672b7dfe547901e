#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_meshgen.py -q -s > gpurun_out/r02k_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02k_pytest.log
