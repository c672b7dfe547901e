#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
RBA_OZAKI=1 timeout 1200 ncu --kernel-name k_oz_gemm --launch-skip 22 --launch-count 1 --set full --import-source on \
  -o gpurun_out/r02h_ozgemm python tools/oz_check.py > gpurun_out/r02h_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02h_ncu.log
