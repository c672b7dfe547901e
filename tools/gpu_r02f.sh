#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -s > gpurun_out/r02f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02f_pytest.log
RBA_OZAKI=1 timeout 600 python tools/oz_check.py > gpurun_out/r02f_oz1.log 2>&1
