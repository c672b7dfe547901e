#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
RBA_OZAKI=0 timeout 600 python tools/oz_check.py > gpurun_out/r02c_oz0.log 2>&1
RBA_OZAKI=1 timeout 600 python tools/oz_check.py > gpurun_out/r02c_oz1.log 2>&1
RBA_OZAKI=1 timeout 900 ncu --kernel-name regex:k_oz --launch-skip 40 --launch-count 4 --set full --import-source on \
  -o gpurun_out/r02c_oz python tools/oz_check.py > gpurun_out/r02c_ncu.log 2>&1
