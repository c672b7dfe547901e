#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_factor_structure.py tests/test_gpu_meshgen.py -q -x > gpurun_out/r02m_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r02m_pytest.log
timeout 600 python tools/oz_check.py > gpurun_out/r02m_oz.log 2>&1
