#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_factor_structure.py tests/test_gpu_ozaki.py tests/test_gpu_verify.py 2>&1 | tail -4
for v in 1 2; do
RBA_FACTOR_STREAMS=$v timeout 600 python tools/oz_check.py > gpurun_out/r02z_oz_s$v.log 2>&1
echo "STREAMS=$v"; grep -h "factor 16" gpurun_out/r02z_oz_s$v.log
done
