#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in 32 64 96 128; do
RBA_LEAF=$v timeout 600 python tools/oz_check.py > gpurun_out/r02z_leaf$v.log 2>&1
echo "LEAF=$v"; grep -h "factor 16\|classes\|^forward" gpurun_out/r02z_leaf$v.log
done
