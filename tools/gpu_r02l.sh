#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/sb_debug.py > gpurun_out/r02l_sb.log 2>&1
timeout 900 python -m pytest tests/test_gpu_meshgen.py -q -s > gpurun_out/r02l_pytest.log 2>&1
timeout 600 python tools/oz_check.py > gpurun_out/r02l_oz.log 2>&1
