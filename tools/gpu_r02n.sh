#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for cfg in "0 4" "1 8" "1 16" "0 8" "1 4"; do
  set -- $cfg
  echo "== trail=$1 panel=$2" >> gpurun_out/r02n.log
  RBA_OZ_TRAIL=$1 RBA_PANEL=$2 timeout 600 python tools/oz_check.py 2>&1 | grep -E "RBA_OZAKI|classes" >> gpurun_out/r02n.log
done
