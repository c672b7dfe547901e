#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_ozaki.py 2>&1 | tail -3
timeout 600 python tools/oz_check.py > gpurun_out/r02z_oz.log 2>&1
grep -h "oz_prof\|factor 16\|classes" gpurun_out/r02z_oz.log
